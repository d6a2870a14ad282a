cd "${GRAFT_REPO_ROOT:-/root/repo}"
export PO_NVCC_EXTRA=-DPO_DIAG
python -c 'from paper_2103_14024_b200 import _build; _build.build()' > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
for r in 1 2; do for cfg in "c1 2" "c1 3" "c3 3" "c3 4" "c1thick 2" "c1thick 3"; do
  set -- $cfg; export PO_RENDER_MINB=$2
  l=$(timeout 600 python bench.py --workload $1 --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | tail -1)
  echo "[$cfg] $(echo "$l" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)"
done; done
