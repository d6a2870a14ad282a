#!/bin/bash
# c4 with the pass-1 group order (costliest first) vs the batch order, interleaved on one box,
# plus the order tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
python -c 'import __graft_entry__ as g; g.build()' > /dev/null 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests/test_gpu_order.py tests/test_gpu_train.py -m gpu -q 2>&1 | tail -2
for r in 1 2; do for o in costliest none; do
  l=$(timeout 900 python bench.py --workload c4 --steps 20 --warmup 5 --pass1-order $o 2>/dev/null | tail -1)
  echo "[$o] r$r $(echo "$l" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e6, d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"]/1e6)' 2>&1 | tail -1)"
done; done
for r in 1 2; do for o in costliest none; do
  l=$(timeout 900 python bench.py --workload c4 --steps 20 --warmup 5 --chunks 4 --unfused-sgd --pass1-order $o 2>/dev/null | tail -1)
  echo "[N>1 path, $o] r$r $(echo "$l" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e6, d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)"
done; done
