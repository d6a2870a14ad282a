cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 compute-sanitizer --tool racecheck --error-exitcode 9 python tools/sanitize_c0.py > gpurun_out/racecheck.log 2>&1; echo "racecheck $?"; tail -3 gpurun_out/racecheck.log
timeout 900 compute-sanitizer --tool synccheck --error-exitcode 9 python tools/sanitize_c0.py > gpurun_out/synccheck.log 2>&1; echo "synccheck $?"; tail -3 gpurun_out/synccheck.log
timeout 900 compute-sanitizer --tool initcheck --error-exitcode 9 python tools/sanitize_c0.py > gpurun_out/initcheck.log 2>&1; echo "initcheck $?"; tail -3 gpurun_out/initcheck.log
VARIANTS="PO_RENDER_OPT=0" bash tools/gpu_ab.sh
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_all.log 2>&1; echo "pytest $?"; tail -2 gpurun_out/pytest_all.log
