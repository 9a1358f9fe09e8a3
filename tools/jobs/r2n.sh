mkdir -p gpurun_out
TAG=r2n
timeout 600 python -m pytest tests -m gpu -q -x -k "packed or race_stress" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 600 python bench.py --steps 3 --warmup 3 --no-latency --no-e2e --no-cpu-baseline --no-pool > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_rc.txt
