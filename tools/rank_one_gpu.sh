#!/bin/bash
# One rank of an N-rank job when only ONE GPU exists (gpurun gives one): every
# rank uses cuda:0, and NCCL_HOSTID differs per rank so NCCL's duplicate-GPU
# check passes -- the ranks then talk over NCCL's socket transport on the
# loopback interface. Exercises the multi-rank code path (torchrun
# rendezvous, NCCL id sharing, the partitioned engine's NCCL send/recv /
# all-gather / broadcast, barriers, max-over-ranks timing); its timings mean
# nothing (N processes share one GPU).
#   python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
#     --master-addr 127.0.0.1 --master-port 29531 --no-python \
#     bash tools/rank_one_gpu.sh bench.py --gpus 2 ...
export NCCL_HOSTID=mglp-rank-$RANK LOCAL_RANK=0 NCCL_SOCKET_IFNAME=lo NCCL_IB_DISABLE=1
exec python "$@"
