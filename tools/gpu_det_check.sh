cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/det; mkdir -p $O
BASE_DIR=ab_base ROUNDS=1 WORKLOADS="c1" TAG=det bash tools/gpu_order_ab2.sh > /dev/null 2>&1
L=paper_2103_14024_b200/libplenoct.so
for v in base new; do
  cp /tmp/lib_$v.so $L; touch $L
  l=$(timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --deterministic --no-cpu-baseline 2>&1 | tail -1)
  echo "[$v] det $(echo "$l" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e6, d["ms_per_step"], d["loss_first_last"])' 2>&1 | tail -1)"
  l=$(timeout 900 python bench.py --workload c4 --steps 5 --warmup 3 --deterministic --pass1-order none --no-cpu-baseline 2>&1 | tail -1)
  echo "[$v] det no-order $(echo "$l" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e6, d["ms_per_step"], d["loss_first_last"])' 2>&1 | tail -1)"
done
cp /tmp/lib_new.so $L; touch $L
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_det.csv python bench.py --workload c4 --steps 2 --warmup 3 --deterministic > /dev/null 2>&1; echo "ncu $?"
