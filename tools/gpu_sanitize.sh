#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over tools/sanitize_c0.py,
# which calls every kernel of libplenoct at c0 sizes.  Outputs: gpurun_out/<tool>.log
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --error-exitcode 9 python tools/sanitize_c0.py > gpurun_out/$tool.log 2>&1
  echo "$tool $?"; tail -2 gpurun_out/$tool.log
done
