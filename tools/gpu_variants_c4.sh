#!/bin/bash
# c4 A/B: VARIANTS="base;-DPO_RAYS_MINB=3" (nvcc flag sets) x BENCH_SETS="|--ray-order tileleaf" (bench args)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
IFS=';' read -ra VS <<< "${VARIANTS:-base}"
IFS='|' read -ra BS <<< "${BENCH_SETS:-}"
[ ${#BS[@]} -eq 0 ] && BS=("")
for v in "${VS[@]}"; do
  [ "$v" = "base" ] && export PO_NVCC_EXTRA="" || export PO_NVCC_EXTRA="$v"
  python -c 'from paper_2103_14024_b200 import _build; _build.build()' > gpurun_out/build_v.log 2>&1 || { echo "BUILD FAILED $v"; continue; }
  for b in "${BS[@]}"; do
    r=$(timeout 900 python bench.py --workload c4 --steps ${STEPS:-20} --warmup 3 $b 2>&1 | tail -1)
    echo "[$v] [$b] $(echo "$r" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"]/1e6,1), d["ms_per_step"], d["loss_first_last"])' 2>&1 | tail -1)"
  done
done
