#!/bin/bash
# c4 after a backward change: full GPU tests, c4 bench lines (fused one-replica step and the
# N>1 code path run at N=1: gradient buffer + 4 chunks), ncu launch list + --set full of the replay
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1800 python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?"; tail -8 gpurun_out/pytest_gpu.log
fi
for v in "" "--chunks 4 --unfused-sgd" ${C4_EXTRA:-}; do
  timeout 900 python bench.py --workload c4 --steps 20 --warmup 3 $v > gpurun_out/c4.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c4.log').read().strip().splitlines()[-1]); print('[$v]', round(d['value']/1e6,1), 'Mrays/s', d['ms_per_step'], 'ms', d['loss_first_last'], d['roofline']['achieved_step'], 'GB/s')" 2>&1 | tail -1
done
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv \
      python bench.py --workload c4 --steps 3 --warmup 3 > /dev/null 2>&1
  echo "ncu launches exit $?"
  timeout 1200 ncu --set full --metrics lts__t_bytes.sum,lts__t_sectors_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum \
      --clock-control none --import-source on --kernel-name-base function -k regex:k_backward_replay_sgd \
      -s 2 -c 1 -f -o gpurun_out/prof_replay python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/ncu_replay.log 2>&1
  echo "ncu replay exit $?"
  timeout 1200 ncu --set full --metrics lts__t_bytes.sum --clock-control none --import-source on --kernel-name-base function \
      -k regex:k_render_rays_p -s 2 -c 1 -f -o gpurun_out/prof_pass1 python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/ncu_pass1.log 2>&1
  echo "ncu pass1 exit $?"
fi
