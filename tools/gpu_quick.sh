cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/s1; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || { echo BUILD FAILED; tail -30 $O/build.log; exit 1; }
timeout 2400 python -m pytest tests -m gpu -q -rs -x > $O/pytest_gpu.log 2>&1; echo "pytest exit $?"; tail -3 $O/pytest_gpu.log
for i in 1 2; do timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_c1_$i.log 2>&1; echo "c1 $?"; tail -1 $O/bench_c1_$i.log; done
for w in c3 c4; do timeout 900 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline > $O/bench_$w.log 2>&1; echo "$w $?"; tail -1 $O/bench_$w.log; done
