cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1 || exit 1
for i in 1 2 3; do for f in write write+read; do
  r=$(timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --flush $f 2>&1 | tail -1)
  echo "[$f] c1 $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["roofline"]["graded"])' 2>&1 | tail -1)"
done; done
for f in write write+read; do
  r=$(timeout 600 python bench.py --workload c3 --steps 20 --warmup 5 --no-cpu-baseline --flush $f 2>&1 | tail -1)
  echo "[$f] c3 $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)"
done
