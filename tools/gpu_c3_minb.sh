cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PO_NVCC_EXTRA=-DPO_DIAG
python -c 'from paper_2103_14024_b200 import _build; _build.build()' > /dev/null 2>&1 || exit 1
for r in 1 2 3; do for m in 3 4; do
  export PO_RENDER_MINB=$m
  l=$(timeout 600 python bench.py --workload c3 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1)
  echo "[c3 minb $m] r$r $(echo "$l" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["frac"])' 2>&1 | tail -1)"
done; done
