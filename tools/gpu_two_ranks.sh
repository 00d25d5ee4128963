#!/bin/bash
# the --gpus N bench path with N ranks on the one GPU (tools/rank_one_gpu.sh)
mkdir -p gpurun_out
TAG=${TAG:-tr}
for n in 2 4; do
  timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n \
    --master-addr 127.0.0.1 --master-port $((29530 + n)) --no-python \
    bash tools/rank_one_gpu.sh bench.py --gpus $n --steps 3 --warmup 3 --extra tiny,mt \
    > gpurun_out/${TAG}_bench_n$n.log 2>&1
  echo "rc=$?" >> gpurun_out/${TAG}_bench_n$n.log
  tail -c 400 gpurun_out/${TAG}_bench_n$n.log
done
grep -h "NET/Socket\|Duplicate\|Using network\|Channel 00" gpurun_out/nccl/*.log 2>/dev/null | head -5
