#!/bin/bash
# The C++ drop-in's master/worker path over P processes on ONE GPU: the
# reference's own launcher (launch_with_master / connect_from_env) starts the
# workers, mmws::gpu::comm_init_from ships the NCCL id over the reference's
# Communicator, and the loopback NCCL stand-in (tests/fake_nccl, test
# infrastructure) carries the exchange.  Gate: bitwise vs mmws::matmul_seq for
# gpu-exact, normwise for gpu-rowblock (the harness's own gate).
#   tools/cpp_world_rehearsal.sh 3 --dims 500,2000 --models gpu-rowblock,gpu-exact
set -e
P=${1:-3}
ROOT=$(cd "$(dirname "$0")/.." && pwd)
LIB=/tmp/libfake_nccl_cpp_rehearsal.so
g++ -std=c++17 -O2 -shared -fPIC -I/usr/local/cuda/include "$ROOT/tests/fake_nccl/fake_nccl.cpp" \
    -o "$LIB" -L/usr/local/cuda/lib64/stubs -lcuda
MMWS_GPU_NCCL_LIB="$LIB" MMWS_BENCH_ONE_GPU_WORLD=1 MMWS_GPU_ROWBLOCK_RANKS=all \
    "$ROOT/oracle/_ref/mmws_gpu_bench_ref" --gpus "$P" "${@:2}"
