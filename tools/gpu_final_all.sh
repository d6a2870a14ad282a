#!/bin/bash
# The whole end-of-round evidence in one call, under gpurun's 64 MiB output limit: tests, smoke,
# every bench line, the 2-rank runs, the diagnostics, the oracle baselines (gpu_final_r02.sh
# with SKIP_NCU=1), then the ncu render captures (c1, c3); the c4 captures are a second call.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${TAG:-final3} SKIP_NCU=1 bash tools/gpu_final_r02.sh
TAG=${TAG:-final3}_ncu PART=render bash tools/gpu_ncu_r02.sh
