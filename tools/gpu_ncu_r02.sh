#!/bin/bash
# ncu captures of the final state, split so each call's gpurun_out stays under 64 MiB:
# PART=render (c1 launch list, --set full of the c1 and c3 frames) or PART=c4 (c4 launch list,
# --set full of the fused replay and of pass 1).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-ncu}; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
X="--metrics lts__t_bytes.sum,lts__t_sectors_op_red.sum,l1tex__t_requests_pipe_lsu_mem_global_op_red.sum"
if [ "${PART:-render}" = render ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c1.csv \
      python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu c1 launches $?"
  timeout 1200 ncu --set full $X --clock-control none --import-source on --kernel-name-base function -k regex:'^k_render$' \
      -s 3 -c 1 -f -o $O/prof_render_c1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu c1 render $?"
  timeout 1200 ncu --set full $X --clock-control none --kernel-name-base function -k regex:'^k_render$' \
      -s 3 -c 1 -f -o $O/prof_render_c3 python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu c3 render $?"
else
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c4.csv \
      python bench.py --workload c4 --steps 3 --warmup 3 > /dev/null 2>&1; echo "ncu c4 launches $?"
  timeout 1200 ncu --set full $X --clock-control none --import-source on --kernel-name-base function -k regex:k_backward_replay_sgd \
      -s 2 -c 1 -f -o $O/prof_replay python bench.py --workload c4 --steps 3 --warmup 3 > /dev/null 2>&1; echo "ncu replay $?"
  timeout 1200 ncu --set full $X --clock-control none --kernel-name-base function -k regex:k_render_rays_p \
      -s 2 -c 1 -f -o $O/prof_pass1 python bench.py --workload c4 --steps 3 --warmup 3 > /dev/null 2>&1; echo "ncu pass1 $?"
fi
du -sh $O
