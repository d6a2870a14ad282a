#!/bin/bash
# A/B: bench under several env settings, one line each. usage: VARIANTS="A=1 B=2;C=3" bash tools/gpu_ab.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
IFS=';' read -ra VS <<< "${VARIANTS:-}"
i=0
for v in "${VS[@]}"; do
  env $v timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS:-} > gpurun_out/ab_$i.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_$i.log').read().strip().splitlines()[-1]); print('[$v]', d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'), d.get('e2e',{}).get('value'))" 2>&1 | tail -1
  i=$((i+1))
done
