#!/bin/bash
# Weak-scaling bench lines at N = 1..NGPU on one box (one rank per GPU, NCCL).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
NG=$(nvidia-smi -L | wc -l)
for n in 1 2 4 8; do
  [ "$n" -gt "$NG" ] && break
  if [ "$n" = 1 ]; then
    timeout 600 python bench.py --gpus 1 ${BENCH_ARGS} > gpurun_out/scale_n1.json 2> gpurun_out/scale_n1.err
  else
    timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 \
      --master-port $((29500 + n)) bench.py --gpus $n ${BENCH_ARGS} > gpurun_out/scale_n$n.json 2> gpurun_out/scale_n$n.err
  fi
  echo "n=$n rc=$?"; cat gpurun_out/scale_n$n.json
done
