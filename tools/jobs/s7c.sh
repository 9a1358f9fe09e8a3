# session 6: stream runner enqueues the LLR upload before building the TTI's tasks: stream-runner parity + cfg5 latency twice
mkdir -p gpurun_out
TAG=${1:-s7c}
timeout 600 python -m pytest tests -m gpu -q -x -k "stream_run or multirank or latency" > gpurun_out/${TAG}_pytest_stream.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
for r in 1 2; do
  timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pool > gpurun_out/${TAG}_lat${r}.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_lat${r}.log').read().strip().splitlines()[-1]);l=d['latency'];i=l['int8_ingest'];print('run$r', 'p50',round(l['p50_us'],1),'p99',round(l['p99_us'],1),'sub',round(l['host_submit_p50_us'],1),'dev',round(l['device_p50_us'],1),'int8',round(i['p50_us'],1),round(i['p99_us'],1), l.get('stages_p50_us'), 'parity', d['parity']['total'])" >> gpurun_out/${TAG}_summary.txt 2>&1
done
