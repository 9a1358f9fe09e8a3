# GPU parity (-x) then a short kernel-only bench
mkdir -p gpurun_out
TAG=${1:-p}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-latency --no-pool > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_rc.txt
