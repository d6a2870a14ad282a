#!/bin/bash
# One gpurun session: build, GPU parity tests, smoke, bench, ncu launch list + full capture.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
if [ "${SKIP_TESTS:-0}" != "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -rs ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest exit $?"; tail -15 gpurun_out/pytest_gpu.log
  timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1
  echo "smoke exit $?"; tail -3 gpurun_out/smoke.log
fi
timeout 900 python bench.py ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1
echo "bench exit $?"; tail -c 3000 gpurun_out/bench.log
if [ "${SKIP_NCU:-0}" != "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
      python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
  echo "ncu launches exit $?"
  timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_render$' \
      -s 3 -c 1 -f -o gpurun_out/prof_render python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
  echo "ncu full exit $?"; tail -5 gpurun_out/ncu_full.log
fi
