#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=final3_c4 PART=c4 bash tools/gpu_ncu_r02.sh
for i in 1 2; do
  l=$(timeout 900 python bench.py --workload c4 --steps 10 --warmup 5 --deterministic --no-cpu-baseline 2>/dev/null | tail -1)
  echo "$l" > gpurun_out/final3_c4/bench_det_$i.log
  echo "[det $i] $(echo "$l" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"]/1e6, d["ms_per_step"], d["e2e"]["value"]/1e6)' 2>&1 | tail -1)"
done
