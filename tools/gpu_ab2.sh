#!/bin/bash
# Interleaved A/B of compile-time variants on one box: VARIANTS="base;-DPO_STEP=1" (semicolon-
# separated nvcc flag sets).  Every variant is built once, then ROUNDS rounds run each variant's
# bench lines back to back (WORKLOADS, default "c1 c3"), so box drift hits every variant alike.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-ab}; mkdir -p $O
L=paper_2103_14024_b200/libplenoct.so
IFS=';' read -ra VS <<< "${VARIANTS:-base}"
i=0
for v in "${VS[@]}"; do
  [ "$v" = "base" ] && export PO_NVCC_EXTRA="" || export PO_NVCC_EXTRA="$v"
  python -c 'from paper_2103_14024_b200 import _build; _build.build()' > $O/build_$i.log 2>&1 || { echo "BUILD FAILED $v"; tail -5 $O/build_$i.log; }
  cp $L /tmp/ab_lib_$i.so; cp $L.flags /tmp/ab_lib_$i.flags; i=$((i+1))
done
for r in $(seq 1 ${ROUNDS:-3}); do
  i=0
  for v in "${VS[@]}"; do
    [ "$v" = "base" ] && export PO_NVCC_EXTRA="" || export PO_NVCC_EXTRA="$v"
    cp /tmp/ab_lib_$i.so $L; cp /tmp/ab_lib_$i.flags $L.flags
    for w in ${WORKLOADS:-c1 c3}; do
      r1=$(timeout 600 python bench.py --workload $w --steps ${STEPS:-20} --warmup 5 --no-cpu-baseline ${BENCH_ARGS:-} 2>$O/err_$i.log | tail -1)
      echo "$r1" >> $O/lines_$i.jsonl
      echo "[$v] r$r $w $(echo "$r1" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d.get("roofline",{}).get("frac"))' 2>&1 | tail -1)"
    done
    i=$((i+1))
  done
done
