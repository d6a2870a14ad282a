#!/bin/bash
# Sweep of the split of the costliest blocks (PO_SPLIT_K blocks, PO_SPLIT_F sub-blocks each) in a
# diagnostics build: c1 and c3 bench lines per setting, ROUNDS interleaved rounds on one box.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-split}; mkdir -p $O
export PO_NVCC_EXTRA=-DPO_DIAG
python -c 'from paper_2103_14024_b200 import _build; _build.build()' > $O/build.log 2>&1 || { echo BUILD FAILED; tail -20 $O/build.log; exit 1; }
for r in $(seq 1 ${ROUNDS:-2}); do
  for kf in ${CONFIGS:-0,1 8,2 16,2 32,2 8,4 16,4 32,4}; do
    export PO_SPLIT_K=${kf%,*} PO_SPLIT_F=${kf#*,}
    for w in ${WORKLOADS:-c1}; do
      l=$(timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>$O/err.log | tail -1)
      echo "$kf $l" >> $O/lines.jsonl
      echo "[K,F=$kf] r$r $w $(echo "$l" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)"
    done
  done
done
