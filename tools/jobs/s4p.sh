# split-path phase-1 pipelining in the latency kernels (+ CRC atomics grouping only for non-uniform warps)
mkdir -p gpurun_out
TAG=${1:-s4p}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_summary.txt
bash tools/jobs/abq.sh ${TAG}q hook pipe
for v in hook pipe; do
  CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_$v.so timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pool --lat-ttis 1000 > gpurun_out/${TAG}_lat_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_lat_$v.log').read().strip().splitlines()[-1]);l=d['latency'];s=d['small_configs'];print('$v', round(l['p50_us'],1), round(l['p99_us'],1), round(l['device_p50_us'],1), 'int8', round(l['int8_ingest']['p50_us'],1), round(l['int8_ingest']['p99_us'],1), 'cfg1', round(s['cfg1']['device_us_p50'],1), 'cfg2', round(s['cfg2']['device_us_p50'],1), l['stages_p50_us'])" >> gpurun_out/${TAG}_summary.txt 2>&1
done
CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_pipe.so CRN_TASK_TRACE_DUMMY=1 true
