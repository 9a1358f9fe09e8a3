mkdir -p gpurun_out
TAG=r2r
timeout 300 python tools/dl_time.py 64 > gpurun_out/${TAG}_dl.json 2>&1
timeout 300 python tools/dl_time.py 256 >> gpurun_out/${TAG}_dl.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
