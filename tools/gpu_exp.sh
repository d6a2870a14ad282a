#!/bin/bash
# experiment run: tests + bench variants (no ncu unless NCU=1)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -rs > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -4 gpurun_out/pytest_gpu.log
fi
for m in ${MINBS:-4}; do
  PO_RENDER_MINB=$m timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/bench_minb$m.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/bench_minb$m.log').read().strip().splitlines()[-1]); print('MINB $m', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])" 2>&1 | tail -1
done
if [ "${NCU:-0}" = "1" ]; then
  PO_RENDER_MINB=${NCU_MINB:-4} timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_render$' \
      -s 3 -c 1 -f -o gpurun_out/prof_render python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
  echo "ncu full exit $?"
fi
