#!/bin/bash
# Multi-GPU round trip (gpurun --gpus N): multi-device parity tests, then the
# bench self-launched at every N this box has.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests -m gpu -x -q -k "multi_device or islands" > gpurun_out/multi_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/multi_pytest.log
tail -3 gpurun_out/multi_pytest.log
for n in 1 2 4 8; do
  [ "$n" -gt "$NG" ] && break
  timeout 900 python bench.py --gpus $n ${BENCH_ARGS} > gpurun_out/multi_n$n.json 2> gpurun_out/multi_n$n.err
  echo "n=$n rc=$?"; cut -c1-400 gpurun_out/multi_n$n.json; grep -c "Init COMPLETE" gpurun_out/multi_n$n.err
done
