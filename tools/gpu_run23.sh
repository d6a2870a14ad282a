cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q > gpurun_out/pytest_full.log 2>&1; echo "fullsize $?"; tail -2 gpurun_out/pytest_full.log
PO_BENCH_BACKEND=gloo PO_BENCH_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 > gpurun_out/bench_2rank.log 2>&1; echo "2rank $?"; tail -c 600 gpurun_out/bench_2rank.log
PO_BENCH_BACKEND=gloo PO_BENCH_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --workload c4 --gpus 2 --steps 4 --warmup 3 --rays 262144 > gpurun_out/c4_2rank.log 2>&1; echo "c4 2rank $?"; tail -c 600 gpurun_out/c4_2rank.log
for o in sampled leaf; do
  timeout 900 python bench.py --workload c4 --steps 10 --warmup 3 --ray-order $o > gpurun_out/c4_$o.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/c4_$o.log').read().strip().splitlines()[-1]); print('c4 $o', d['value'], d['ms_per_step'], d['loss_first_last'])"
done
timeout 900 compute-sanitizer --tool memcheck --error-exitcode 9 python tools/sanitize_c0.py > gpurun_out/memcheck.log 2>&1; echo "memcheck $?"; tail -4 gpurun_out/memcheck.log
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_c0.py > gpurun_out/racecheck.log 2>&1; echo "racecheck $?"; tail -4 gpurun_out/racecheck.log
