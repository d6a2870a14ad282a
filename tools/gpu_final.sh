#!/bin/bash
# End-of-round evidence in one gpurun call: tests + smoke + c1 bench + ncu (gpu_check.sh), the
# c2 / c3 / c4 bench lines, the N=2 paths and the sanitizers.  Outputs under gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
bash tools/gpu_check.sh > gpurun_out/final_check.log 2>&1
tail -12 gpurun_out/final_check.log | cut -c1-200
for w in c2 c3 c4; do
  timeout 900 python bench.py --workload $w --steps ${STEPS:-50} > gpurun_out/final_$w.log 2>&1
  echo "$w exit $?"; tail -1 gpurun_out/final_$w.log | cut -c1-160
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_c4_launches.csv \
    python bench.py --workload c4 --steps 3 --warmup 3 > /dev/null 2>&1; echo "ncu c4 launches $?"
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:k_backward_replay \
    -s 2 -c 1 -f -o gpurun_out/final_prof_replay python bench.py --workload c4 --steps 3 --warmup 3 > /dev/null 2>&1
echo "ncu replay $?"
bash tools/gpu_multirank.sh 2>&1 | grep exit
bash tools/gpu_sanitize.sh 2>&1 | grep -E "^(memcheck|racecheck|synccheck|initcheck)"
