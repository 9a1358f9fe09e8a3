mkdir -p gpurun_out
TAG=${1:-rm}
timeout 600 python -m pytest tests -m gpu -q -k "rate or encode or chain" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-latency --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_rc.txt
