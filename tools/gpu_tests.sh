#!/bin/bash
# build + the GPU test suite (+ smoke); PYTEST_K selects tests (pytest -k expression)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
if [ -n "${PYTEST_K:-}" ]; then
  timeout ${PYTEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q -rs -x -k "$PYTEST_K" > gpurun_out/pytest_gpu.log 2>&1
else
  timeout ${PYTEST_TIMEOUT:-1800} python -m pytest tests -m gpu -q -rs -x > gpurun_out/pytest_gpu.log 2>&1
fi
echo "pytest exit $?"; tail -25 gpurun_out/pytest_gpu.log
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1
echo "smoke exit $?"; tail -3 gpurun_out/smoke.log
