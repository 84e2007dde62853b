#!/bin/bash
# Rehearse the N=2 bench control flow on ONE GPU: both ranks on cuda:0, gloo for
# torch.distributed plumbing, CUDA IPC for the KV migration — one-sided pull, or
# TRANSPORT=push (the prefill kernel stores the pages into the decoder's mapped
# pool) — since NCCL refuses two ranks on one GPU. NOT a performance measurement.
export CUDA_VISIBLE_DEVICES=0
python -m torch.distributed.run --nnodes=1 --nproc-per-node ${NPROC:-2} --master-addr 127.0.0.1 --master-port 29611 \
  tools/local_rank0.py bench.py --gpus ${NPROC:-2} --steps 2 --warmup 2 --batch 4 --no-cpu-baseline \
  --transport ${TRANSPORT:-pull} --pg-backend gloo "$@"
