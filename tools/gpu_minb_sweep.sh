cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/minb; mkdir -p $O
export PO_NVCC_EXTRA=-DPO_DIAG
python -c 'from paper_2103_14024_b200 import _build; _build.build()' > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python tools/timeline_view.py c3 > $O/tl_c3.txt 2>&1; cat $O/tl_c3.txt
python tools/timeline_view.py c1 > $O/tl_c1.txt 2>&1; cat $O/tl_c1.txt
for r in 1 2; do
for cfg in "c1 2 8 2" "c1 3 8 2" "c1 3 16 2" "c1 3 32 4" "c3 2 8 2" "c3 3 8 2" "c3 4 8 2"; do
  set -- $cfg
  export PO_RENDER_MINB=$2 PO_SPLIT_K=$3 PO_SPLIT_F=$4
  l=$(timeout 600 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu-baseline 2>$O/err.log | tail -1)
  echo "[$cfg] $(echo "$l" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)"
done
done
