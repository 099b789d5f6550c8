#!/bin/bash
# A/B: headline bench (device-resident eval only) for the default build and
# each variant library given as build/<name>/libhetsched_sm100a.so.
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
mkdir -p gpurun_out
ARGS=${AB_ARGS:---steps 10 --warmup 3 --no-ga --no-sweep --no-cpu-baseline}
echo "default: $(timeout 300 python bench.py $ARGS 2>gpurun_out/ab_default.err | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["kernel_ms"], d["clocks"])')"
for v in "$@"; do
  echo "$v: $(HS_LIB_PATH=build/$v/libhetsched_sm100a.so timeout 300 python bench.py $ARGS 2>gpurun_out/ab_$v.err | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(d["value"], d["roofline"]["kernel_ms"], d["clocks"])')"
done
