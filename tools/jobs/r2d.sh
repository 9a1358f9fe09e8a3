# round-2 evidence run: smoke, full pytest -m gpu, default bench line (each under its own timeout)
mkdir -p gpurun_out
TAG=${1:-r2d}
nvidia-smi > gpurun_out/${TAG}_nvsmi.txt 2>&1; nproc >> gpurun_out/${TAG}_nvsmi.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=20 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 700 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_rc.txt
