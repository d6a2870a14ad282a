#!/bin/bash
# A/B of compile-time variants: VARIANTS="-DPO_ECACHE=1;-DPO_EVICT=1" (semicolon-separated nvcc
# flag sets; "base" = none).  Each variant: build, c1 bench (20/5) twice, c3 bench once.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-base}"
for v in "${VS[@]}"; do
  [ "$v" = "base" ] && export PO_NVCC_EXTRA="" || export PO_NVCC_EXTRA="$v"
  python -c 'from paper_2103_14024_b200 import _build; _build.build()' > gpurun_out/build_v.log 2>&1 || { echo "BUILD FAILED $v"; tail -5 gpurun_out/build_v.log; continue; }
  for w in ${WORKLOADS:-c1 c1 c3}; do
    r=$(timeout 600 python bench.py --workload $w --steps ${STEPS:-40} --warmup 5 --no-cpu-baseline 2>&1 | tail -1)
    echo "[$v] $w $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"])' 2>&1 | tail -1)"
  done
done
