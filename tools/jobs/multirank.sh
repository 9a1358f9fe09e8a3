# functional check of bench.py's N > 1 path on a one-GPU box: 2 ranks, gloo, both on cuda:0
# (ranks never wait on each other's kernels; the line carries functional_check_only)
mkdir -p gpurun_out
TAG=${1:-mr}
for SC in weak strong; do
CRN_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
    --master-addr 127.0.0.1 --master-port 29531 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo \
    --scaling $SC > gpurun_out/${TAG}_${SC}.log 2>&1; echo "multirank $SC rc=$?" >> gpurun_out/${TAG}_rc.txt
done
