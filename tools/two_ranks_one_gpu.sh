#!/bin/bash
# Rehearse the N=2 bench control flow on ONE GPU: both ranks on cuda:0, gloo for
# torch.distributed plumbing, one-sided CUDA-IPC pull for the KV migration (NCCL
# refuses two ranks on one GPU). NOT a performance measurement.
export CUDA_VISIBLE_DEVICES=0
python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NPROC:-2} --master-addr 127.0.0.1 --master-port 29611 \
  tools/local_rank0.py bench.py --gpus ${NPROC:-2} --steps 2 --warmup 2 --batch 4 --no-cpu-baseline \
  --transport pull --pg-backend gloo "$@"
