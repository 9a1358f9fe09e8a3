# A/B: group tasks packed three per CTA (grid = CTA units) vs spread one per CTA (CRN_GRID_SPREAD=1)
mkdir -p gpurun_out
TAG=${1:-s4c}
for r in 1 2; do
  timeout 200 python tools/ab_quick.py --tag packed --save /tmp/abq_packed.pt >> gpurun_out/${TAG}_summary.txt 2>> gpurun_out/${TAG}_err.txt
  CRN_GRID_SPREAD=1 timeout 200 python tools/ab_quick.py --tag spread --ref /tmp/abq_packed.pt >> gpurun_out/${TAG}_summary.txt 2>> gpurun_out/${TAG}_err.txt
done
for m in 0 1; do
  CRN_GRID_SPREAD=$m timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pool --lat-ttis 500 > gpurun_out/${TAG}_lat$m.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_lat$m.log').read().strip().splitlines()[-1]);l=d['latency'];s=d['small_configs'];print('spread=$m', round(l['p50_us'],1), round(l['p99_us'],1), round(l['device_p50_us'],1), 'int8', round(l['int8_ingest']['p50_us'],1), round(l['int8_ingest']['p99_us'],1), 'cfg1', round(s['cfg1']['device_us_p50'],1), 'cfg2', round(s['cfg2']['device_us_p50'],1))" >> gpurun_out/${TAG}_summary.txt 2>&1
done
