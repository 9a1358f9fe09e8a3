# A/B incl. small configs and TTI latency: variants/libcrn_<v>.so
mkdir -p gpurun_out
TAG=${1:-abl}
shift
for v in "$@"; do
  CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_$v.so timeout 600 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --lat-ttis 400 > gpurun_out/${TAG}_$v.log 2>&1
  python -c "import json;d=json.loads(open('gpurun_out/${TAG}_$v.log').read().strip().splitlines()[-1]);s=d['small_configs'];l=d['latency'];print('$v', round(d['ms_per_step'],3), round(s['cfg1']['device_us_p50'],1), round(s['cfg2']['device_us_p50'],1), round(l['p50_us'],1), round(l['p99_us'],1), round(d['pool_tti']['decode_ms'],3))" >> gpurun_out/${TAG}_summary.txt 2>&1
done
