# session-4 final evidence: smoke, GPU tests, default bench line, reference arm, decode launch list
mkdir -p gpurun_out
TAG=${1:-s4r}
nvidia-smi > gpurun_out/${TAG}_nvsmi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_ref.log 2>&1; echo "ref rc=$?" >> gpurun_out/${TAG}_rc.txt
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/${TAG}_rc.txt
