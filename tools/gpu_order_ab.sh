cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/s5; mkdir -p $O
python -c 'import __graft_entry__ as g; g.build()' > $O/build.log 2>&1 || { echo BUILD FAILED; tail -30 $O/build.log; exit 1; }
for r in 1 2; do
for mode in adaptive centre; do
  for w in c1 c3; do
    if [ $mode = centre ]; then export PO_RENDER_ORDER=centre; else unset PO_RENDER_ORDER; fi
    l=$(timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>$O/err.log | tail -1)
    echo "$l" >> $O/lines_$mode.jsonl
    echo "[$mode] $w $(echo "$l" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"])' 2>&1 | tail -1)"
  done
done
done
unset PO_RENDER_ORDER
timeout 1500 python -m pytest tests -m gpu -q -x > $O/pytest.log 2>&1; echo "pytest $?"; tail -3 $O/pytest.log
