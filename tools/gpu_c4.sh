#!/bin/bash
# c4 optimisation-step measurements + ncu of the backward kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
for a in "${C4_VARIANTS:---lr 1e-4}"; do :; done
IFS=';' read -ra VS <<< "${C4_VARIANTS:---lr 1e-4}"
i=0
for v in "${VS[@]}"; do
  timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 $v > gpurun_out/c4_$i.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c4_$i.log').read().strip().splitlines()[-1]); print('[$v]', d['value'], d['ms_per_step'], d['loss_first_last'], d['roofline']['achieved_step'])" 2>&1 | tail -1
  i=$((i+1))
done
if [ "${NCU:-1}" = "1" ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4_launches.csv \
      python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/c4_ncu_launches.log 2>&1
  echo "ncu launches exit $?"
  timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_backward$' \
      -s 3 -c 1 -f -o gpurun_out/prof_backward python bench.py --workload c4 --steps 3 --warmup 3 > gpurun_out/ncu_bwd.log 2>&1
  echo "ncu bwd exit $?"
fi
