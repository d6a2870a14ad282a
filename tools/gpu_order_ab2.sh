#!/bin/bash
# A/B of two builds (BASE_REF = git ref of the base; the working tree is the candidate):
# c1 and c3 bench lines, ROUNDS interleaved rounds on one box, then the order tests.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
O=gpurun_out/${TAG:-ab2}; mkdir -p $O
L=paper_2103_14024_b200/libplenoct.so
python -c 'from paper_2103_14024_b200 import _build; _build.build()' > $O/build_new.log 2>&1 || { echo BUILD FAILED; exit 1; }
cp $L /tmp/lib_new.so
cp -r paper_2103_14024_b200/csrc /tmp/csrc_new
git_base=${BASE_DIR:-}
if [ -n "$git_base" ]; then
  cp $git_base/*.cu $git_base/*.cuh $git_base/*.h paper_2103_14024_b200/csrc/
  python -c 'from paper_2103_14024_b200 import _build; _build.build(force=True)' > $O/build_base.log 2>&1 || { echo BASE BUILD FAILED; exit 1; }
  cp $L /tmp/lib_base.so
  cp /tmp/csrc_new/* paper_2103_14024_b200/csrc/
fi
for r in $(seq 1 ${ROUNDS:-2}); do
  for v in base new; do
    [ -f /tmp/lib_$v.so ] || continue
    cp /tmp/lib_$v.so $L; touch $L
    for w in ${WORKLOADS:-c1 c3}; do
      l=$(timeout 600 python bench.py --workload $w --steps 20 --warmup 5 --no-cpu-baseline 2>$O/err.log | tail -1)
      echo "$v $l" >> $O/lines.jsonl
      echo "[$v] r$r $w $(echo "$l" | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["ms_per_step"], d["roofline"]["frac"], d["e2e"]["value"])' 2>&1 | tail -1)"
    done
  done
done
cp /tmp/lib_new.so $L; touch $L
