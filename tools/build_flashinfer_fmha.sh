#!/bin/bash
# Build flashinfer's trtllm-gen FMHA launcher (JIT module, library code used only by
# tools/library_baselines.py) on the CPU host into .fi_ws/ (git-ignored, travels with
# gpurun); on the box export the same two variables before running the baselines.
set -e
cd "$(dirname "$0")/.."
export FLASHINFER_WORKSPACE_BASE=$PWD/.fi_ws FLASHINFER_CUDA_ARCH_LIST=10.0a
python -c "from flashinfer.jit.attention.modules import gen_trtllm_gen_fmha_module as g; m = g(); m.build(verbose=False); print(m.get_library_path())"
