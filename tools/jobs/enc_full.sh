mkdir -p gpurun_out
TAG=${1:-encf}
B="python bench.py --steps 1 --warmup 3 --no-latency --no-e2e --no-cpu-baseline"
timeout 900 ncu --set full --clock-control none --import-source on -k encode_kernel -s 1 -c 1 -o gpurun_out/${TAG}_encode $B > gpurun_out/${TAG}_1.log 2>&1; echo "e rc=$?" >> gpurun_out/${TAG}_rc.txt
