mkdir -p gpurun_out
TAG=${1:-rmn}
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"match|encode" --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 1 --warmup 3 --no-latency --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_rc.txt
