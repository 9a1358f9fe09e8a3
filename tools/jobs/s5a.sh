# session 5: stream-runner completion by host flag (cuStreamWriteValue32) vs event polling (CRN_STREAM_EVQ=1)
mkdir -p gpurun_out
TAG=${1:-s5a}
timeout 600 python -m pytest tests -m gpu -q -x -k "stream_run or multirank" > gpurun_out/${TAG}_pytest_stream.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
for r in 1 2; do
  for v in flag evq; do
    if [ $v = evq ]; then export CRN_STREAM_EVQ=1; else unset CRN_STREAM_EVQ; fi
    timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --no-pool > gpurun_out/${TAG}_${v}${r}.log 2>&1
    python -c "import json;d=json.loads(open('gpurun_out/${TAG}_${v}${r}.log').read().strip().splitlines()[-1]);l=d['latency'];i=l['int8_ingest'];print('$v$r', 'p50',round(l['p50_us'],1),'p99',round(l['p99_us'],1),'sub',round(l['host_submit_p50_us'],1),'dev',round(l['device_p50_us'],1),'int8',round(i['p50_us'],1),round(i['p99_us'],1), l.get('stages_p50_us'))" >> gpurun_out/${TAG}_summary.txt 2>&1
  done
done
unset CRN_STREAM_EVQ
