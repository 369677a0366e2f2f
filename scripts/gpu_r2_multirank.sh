#!/usr/bin/env bash
# The bench's multi-rank code path (peer-memory sharding, max-over-ranks
# timing, rank-0 JSON) with two ranks sharing the one GPU over gloo.
cd "${GRAFT_REPO_ROOT:-.}"
mkdir -p gpurun_out
for w in tcf gqf gqf_kmer bulk_tcf; do
  FK_BENCH_BACKEND=gloo timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --workload $w --log-slots 24 --no-cpu > gpurun_out/r2mr_$w.json 2> gpurun_out/r2mr_$w.err; echo "$w rc=$?"
  tail -c 600 gpurun_out/r2mr_$w.json; tail -3 gpurun_out/r2mr_$w.err
done
