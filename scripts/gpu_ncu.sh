#!/bin/bash
# ncu evidence for the eval kernel: launch list + one full capture (1 GPU).
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
TAG=${TAG:-prof}
CMD="python bench.py --population ${NCU_P:-1048576} --steps 3 --warmup 3 --no-cpu-baseline"
$CMD > gpurun_out/${TAG}_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-eval_warp} -s ${NCU_SKIP:-3} -c 1 -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
echo "rc=$?"
tail -3 gpurun_out/${TAG}_plain.log; tail -5 gpurun_out/${TAG}_ncu_full.log
