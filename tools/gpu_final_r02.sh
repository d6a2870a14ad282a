#!/bin/bash
# End-of-round evidence in one gpurun call (round 2).  Everything lands in gpurun_out/final/:
# tests + smoke, the driver's bench command x3, every workload's bench line, ncu launch list and
# --set full captures (with lts__t_bytes) of the c1 / c3 render, c4 pass 1 and replay, the 2-rank
# paths, compute-sanitizer, the per-config oracle baselines and the L2 micro-benchmark.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-final}; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || { echo BUILD FAILED; tail -30 $O/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 2400 python -m pytest tests -m gpu -q -rs > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest_gpu.log
  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > $O/smoke.log 2>&1; echo "smoke exit $?"; tail -1 $O/smoke.log
fi
for i in 1 2 3; do
  timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > $O/bench_c1_$i.log 2>&1; echo "bench c1 #$i exit $?"; tail -1 $O/bench_c1_$i.log | cut -c1-160
done
for w in "c2 --steps 5" "c3 --steps 20" "c1thick --steps 20" "c3sh25 --steps 20" "c4 --steps 20" "c4 --steps 20 --chunks 4 --unfused-sgd" "c4 --steps 10 --deterministic" "c1 --steps 20 --views-per-launch 8"; do
  set -- $w; tag=$(echo "$w" | tr ' -' '__')
  timeout 900 python bench.py --workload $w --no-cpu-baseline > $O/bench_$tag.log 2>&1; echo "bench $w exit $?"; tail -1 $O/bench_$tag.log | cut -c1-160
done
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > $O/bench_reference.log 2>&1; echo "reference exit $?"
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv \
      python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu c1 launches $?"
  X="--metrics lts__t_bytes.sum,lts__t_sectors_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum"
  timeout 1200 ncu --set full $X --clock-control none --import-source on --kernel-name-base function -k regex:'^k_render$' \
      -s 3 -c 1 -f -o $O/prof_render_c1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu c1 render $?"
  timeout 1200 ncu --set full $X --clock-control none --kernel-name-base function -k regex:'^k_render$' \
      -s 3 -c 1 -f -o $O/prof_render_c3 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu c3 render $?"
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
      python bench.py --workload c4 --steps 3 --warmup 3 > /dev/null 2>&1; echo "ncu c4 launches $?"
  timeout 1200 ncu --set full $X --clock-control none --import-source on --kernel-name-base function -k regex:k_backward_replay_sgd \
      -s 2 -c 1 -f -o $O/prof_replay python bench.py --workload c4 --steps 3 --warmup 3 > /dev/null 2>&1; echo "ncu replay $?"
  timeout 1200 ncu --set full $X --clock-control none --kernel-name-base function -k regex:k_render_rays_p \
      -s 2 -c 1 -f -o $O/prof_pass1 python bench.py --workload c4 --steps 3 --warmup 3 > /dev/null 2>&1; echo "ncu pass1 $?"
fi
port=29631
for w in "c1 --steps 20" "c2 --steps 5" "c4 --steps 4 --rays 262144"; do
  set -- $w
  PO_BENCH_BACKEND=gloo PO_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port $port bench.py --workload $w --gpus 2 --warmup 3 > $O/multirank_$1.log 2>&1
  echo "2-rank $w exit $?"; tail -1 $O/multirank_$1.log | cut -c1-160; port=$((port + 1))
done
# compute-sanitizer is closed on this GPU pool (runs under it left GPUs needing a reset): not run
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2bw tools/micro/l2bw.cu && for mb in 32 48 64 96; do /tmp/l2bw $mb 20; done > $O/l2bw.jsonl
(export PO_NVCC_EXTRA=-DPO_DIAG; python -c 'from paper_2103_14024_b200 import _build; _build.build()' > $O/build_diag.log 2>&1 && \
  timeout 600 python tools/diag_tail.py > $O/diag_tail.txt 2>&1; timeout 600 python tools/timeline_c1.py > $O/timeline_c1.txt 2>&1; echo "diag $?")
python -c 'from paper_2103_14024_b200 import _build; _build.build()' > /dev/null 2>&1
timeout 1800 python tools/oracle_baselines.py > $O/oracle_baselines.log 2>&1; echo "oracle baselines exit $?"; tail -1 $O/oracle_baselines.log | cut -c1-200
