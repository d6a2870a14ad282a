cd "${GRAFT_REPO_ROOT:-/root/repo}"
SKIP_NCU=1 bash tools/gpu_check.sh
timeout 600 python bench.py --workload c4 --steps 10 --warmup 3 > gpurun_out/bench_c4.log 2>&1; echo "c4 exit $?"; tail -c 2500 gpurun_out/bench_c4.log
timeout 1200 ncu --set full --clock-control none --import-source on --kernel-name-base function -k regex:'^k_render$' \
      -s 3 -c 1 -f -o gpurun_out/prof_render python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
echo "ncu full exit $?"
