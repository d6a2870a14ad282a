#!/bin/bash
# A/B of c4 variants: usage VARIANTS="A=1;B=2" bash tools/gpu_ab_c4.sh
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
IFS=';' read -ra VS <<< "${VARIANTS:-}"
i=0
for v in "${VS[@]}"; do
  env $v timeout 600 python bench.py --workload c4 --steps ${STEPS:-30} ${BENCH_ARGS:-} > gpurun_out/abc4_$i.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/abc4_$i.log').read().strip().splitlines()[-1]); print('[$v]', round(d['value']/1e6,1), d['ms_per_step'], round(d['e2e']['value']/1e6,1), d['loss_first_last'])" 2>&1 | tail -1
  i=$((i+1))
done
