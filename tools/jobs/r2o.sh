mkdir -p gpurun_out
TAG=r2o
timeout 900 python -m pytest tests -m gpu -q -x -k "packed or race_stress" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_trace.so timeout 300 python tools/task_trace.py 5 6 > gpurun_out/${TAG}_trace_cfg5.json 2> gpurun_out/${TAG}_trace_err.txt
CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_trace.so timeout 300 python tools/task_trace.py 3 1 > gpurun_out/${TAG}_trace_cfg3.json 2>> gpurun_out/${TAG}_trace_err.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-latency --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_rc.txt
