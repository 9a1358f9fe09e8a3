# parity + bench + ncu launch list + one full capture of the decode kernel
mkdir -p gpurun_out
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
timeout 600 $B > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launches.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/rc.txt
B1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B1 > gpurun_out/plain1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
    -o gpurun_out/prof_decode $B1 > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/rc.txt
