mkdir -p gpurun_out
TAG=${1:-li}
for G in 1 2 4; do
  timeout 600 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-pool --lat-ttis 1000 --lat-groups $G > gpurun_out/${TAG}_$G.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_$G.log').read().strip().splitlines()[-1]);l=d['latency'];e=l['int8_ingest'];print($G, 'int16', round(l['p50_us'],1), round(l['p99_us'],1), 'int8', round(e['p50_us'],1), round(e['p99_us'],1))" >> gpurun_out/${TAG}_summary.txt 2>&1
done
