mkdir -p gpurun_out
TAG=r2j
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
B1="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-latency --no-pool"
CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_bulk.so timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 3 -c 1 \
    -o gpurun_out/${TAG}_bulk $B1 > gpurun_out/${TAG}_ncu_bulk.log 2>&1; echo "ncu rc=$?" >> gpurun_out/${TAG}_rc.txt
