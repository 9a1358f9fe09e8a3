# functional check of bench.py's N-rank path on one GPU (gloo, all ranks on cuda:0):
# N = 4 and 8, weak scaling, no e2e (each rank would pin 2.4 GB of host LLRs)
mkdir -p gpurun_out
TAG=${1:-mrn}
for N in 4 8; do
CRN_BENCH_SHARE_GPU=1 timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 2953$N bench.py --gpus $N --steps 2 --warmup 3 --dist-backend gloo \
    --no-e2e > gpurun_out/${TAG}_$N.log 2>&1; echo "multirank N=$N rc=$?" >> gpurun_out/${TAG}_rc.txt
done
