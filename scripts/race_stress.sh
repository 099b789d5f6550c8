#!/bin/bash
# Race stress in place of compute-sanitizer (closed on the GPU pool): a
# library built with -DHS_RACE_JITTER (random per-thread sleeps at every
# cross-warp / cross-CTA hand-off, hs_common.cuh) must still reproduce the
# oracle bit for bit on the race-prone kernels: eval8 Held-Karp set sharing,
# the cluster Held-Karp async-push layers, the streamed host-path kernel
# (chunk arrival / finished counts), GA sweep waves and island syncs.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
export HS_LIB_PATH=build/jitter/libhetsched_sm100a.so
for rep in 1 2 3; do
  timeout 900 python scripts/sanitize_probe.py > gpurun_out/race_probe_$rep.log 2>&1; echo "probe rep $rep rc=$?"
done
timeout 1500 python -m pytest tests -m gpu -x -q -k "20k or cluster or evolve_1000 or islands or warp_island or two_streams or multi_device or golden or streamed or spans or batch_priced or large_device or config45" \
  > gpurun_out/race_pytest.log 2>&1; echo "pytest rc=$?"
tail -2 gpurun_out/race_pytest.log; tail -1 gpurun_out/race_probe_1.log
