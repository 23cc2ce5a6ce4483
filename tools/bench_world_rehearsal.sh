#!/bin/bash
# Rehearsal of the driver's N-GPU bench line on ONE GPU: bench.py --gpus N at its
# default sizes with every rank on GPU 0 through the loopback NCCL stand-in
# (tests/fake_nccl, test infrastructure).  Exercises the full N>1 code path of
# bench.py and the engine; the times measure nothing about NVLink.
#   tools/bench_world_rehearsal.sh 8 > gpurun_out/rehearsal8.json
set -e
N=${1:-8}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
LIB=/tmp/libfake_nccl_rehearsal.so
g++ -std=c++17 -O2 -shared -fPIC -I/usr/local/cuda/include "$ROOT/tests/fake_nccl/fake_nccl.cpp" \
    -o "$LIB" -L/usr/local/cuda/lib64/stubs -lcuda
env -u RANK -u WORLD_SIZE -u LOCAL_RANK -u MASTER_ADDR -u MASTER_PORT \
    MMWS_GPU_NCCL_LIB="$LIB" MMWS_BENCH_ONE_GPU_WORLD=1 \
    python "$ROOT/bench.py" --gpus "$N" "${@:2}"
