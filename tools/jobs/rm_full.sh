mkdir -p gpurun_out
TAG=${1:-rmf}
B="python bench.py --steps 1 --warmup 3 --no-latency --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k match_kernel -c 1 -o gpurun_out/${TAG}_match $B > gpurun_out/${TAG}_1.log 2>&1; echo "m rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k dematch_kernel -c 1 -o gpurun_out/${TAG}_dematch $B > gpurun_out/${TAG}_2.log 2>&1; echo "d rc=$?" >> gpurun_out/${TAG}_rc.txt
