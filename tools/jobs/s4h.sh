# latency kernels (rolled phase 1, one SISO call site): parity both ways + A/B timing
mkdir -p gpurun_out
TAG=${1:-s4h}
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_summary.txt
CRN_ROLL=1 timeout 900 python -m pytest tests -m gpu -x -q -k "not cfg4_full and not multirank" > gpurun_out/${TAG}_pytest_roll1.log 2>&1; echo "pytest roll=1 rc=$?" >> gpurun_out/${TAG}_summary.txt
bash tools/jobs/abq.sh ${TAG}q s roll
for v in s roll; do
  CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_$v.so timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pool --lat-ttis 500 > gpurun_out/${TAG}_lat_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_lat_$v.log').read().strip().splitlines()[-1]);l=d['latency'];print('$v', round(l['p50_us'],1), round(l['p99_us'],1), round(l['device_p50_us'],1), 'int8', round(l['int8_ingest']['p50_us'],1), round(l['int8_ingest']['p99_us'],1), l['stages_p50_us'])" >> gpurun_out/${TAG}_summary.txt 2>&1
done
