#!/bin/bash
# compute-sanitizer passes over one small fused IMEX step (the smoke case: 144 columns x 8 layers,
# every stepper kernel incl. the cp.async rings, tile staging and the block-Thomas workspace) and
# the peer-store halo on virtual ranks.  Output: gpurun_out/sanitize/<tool>.log
set -u
mkdir -p gpurun_out/sanitize
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 \
      python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize/$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize/summary.txt
done
timeout 1200 $CS --tool memcheck --print-limit 20 --error-exitcode 9 \
    python -m pytest -q tests/test_partition_gpu.py -k "peer_store and 2" > gpurun_out/sanitize/memcheck_p2p.log 2>&1
echo "memcheck p2p rc=$?" >> gpurun_out/sanitize/summary.txt
