# session-4 evidence: smoke, default bench line, decode launch list, ncu full capture of the CRC-ET kernel on cfg3
mkdir -p gpurun_out
TAG=${1:-s4m}
nvidia-smi > gpurun_out/${TAG}_nvsmi.txt 2>&1
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_rc.txt
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 300 python tools/small_decode.py 3 > gpurun_out/${TAG}_plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 \
    -o gpurun_out/${TAG}_cfg3 python tools/small_decode.py 3 > gpurun_out/${TAG}_ncu3.log 2>&1; echo "ncu cfg3 rc=$?" >> gpurun_out/${TAG}_rc.txt
