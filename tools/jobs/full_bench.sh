# smoke + GPU tests + the default bench line (e2e, latency, cpu_baseline included)
mkdir -p gpurun_out
TAG=${1:-fb}
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/${TAG}_rc.txt
