mkdir -p gpurun_out
TAG=r2q
bash tools/jobs/abq.sh ${TAG}_ab hd1 sp hd1 sp
CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_trace_sp.so timeout 300 python tools/task_trace.py 5 6 > gpurun_out/${TAG}_trace_cfg5.json 2> gpurun_out/${TAG}_trace_err.txt
timeout 900 python -m pytest tests -m gpu -q -x -k "packed or race_stress or every_k or many_small or group_tasks" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 900 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --lat-ttis 300 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_rc.txt
