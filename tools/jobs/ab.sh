# A/B: time each paper_1905_01141_b200/variants/libcrn_<v>.so on the bench (kernel only)
mkdir -p gpurun_out
TAG=${1:-ab}
shift
for v in "$@"; do
  for r in 1 2; do
    CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_$v.so timeout 300 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-latency --no-pool > gpurun_out/${TAG}_$v$r.log 2>&1
    python -c "import json;d=json.load(open('gpurun_out/${TAG}_$v$r.log'));print('$v', d['ms_per_step'], round(d['roofline']['frac'],4))" >> gpurun_out/${TAG}_summary.txt 2>&1
  done
done
