#!/bin/bash
# The N>1 bench paths on a one-GPU box: 2 ranks with gloo, both pinned to device 0
# (PO_BENCH_BACKEND / PO_BENCH_DEVICE, bench.py _dist).  Exercises view sharding (c1, c2) and
# the data-parallel optimisation step with the chunked pass-2 / allreduce overlap (c4).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c 'import __graft_entry__ as g; g.build()' > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
port=29611
for wl in "c1 --steps 20" "c1 --steps 20 --shard tile" "c2 --steps 5" "c4 --steps 4 --rays 262144"; do
  set -- $wl
  PO_BENCH_BACKEND=gloo PO_BENCH_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
      --master-addr 127.0.0.1 --master-port $port bench.py --workload $wl --gpus 2 --warmup 3 \
      > gpurun_out/multirank_$1$3$4.log 2>&1
  echo "$wl 2-rank exit $?"; tail -1 gpurun_out/multirank_$1$3$4.log | cut -c1-240
  port=$((port + 1))
done


# reduce-scatter vs allreduce (bitwise): tests/test_gpu_multirank.py
