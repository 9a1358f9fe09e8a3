# usage: bash tools/jobs/prof.sh <tag>   -- launch list + one full capture of the decode kernel
mkdir -p gpurun_out
TAG=${1:-prof}
B="python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B > gpurun_out/${TAG}_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "timed/" --csv \
    --log-file gpurun_out/${TAG}_launches.csv $B > gpurun_out/${TAG}_ncu_launches.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/rc.txt
B1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
timeout 600 $B1 > gpurun_out/${TAG}_plain1.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG} $B1 > gpurun_out/${TAG}_ncu_full.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/rc.txt
