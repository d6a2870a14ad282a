cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q -rs -k "descends or optimizer" > gpurun_out/pytest_opt.log 2>&1; echo "pytest $?"; grep -E "passed|failed|assert|losses" gpurun_out/pytest_opt.log | head -10
timeout 900 python bench.py --workload c3 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "c3 $?"; tail -c 1500 gpurun_out/bench_c3.log
for v in "--ray-sampling tile --lr 1e-4" "--ray-sampling tile --lr 3" "--ray-sampling pixel --lr 1e-4"; do
  timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 $v > gpurun_out/c4v.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c4v.log').read().strip().splitlines()[-1]); print('[$v]', d['value'], d['ms_per_step'], d['loss_first_last'])" 2>&1 | tail -1
done
