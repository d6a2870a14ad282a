cd "${GRAFT_REPO_ROOT:-/root/repo}"
BASE_DIR=ab_base ROUNDS=2 WORKLOADS="c3sh25" TAG=sh25 bash tools/gpu_order_ab2.sh
TAG=ncu_c4 PART=c4 bash tools/gpu_ncu_r02.sh
