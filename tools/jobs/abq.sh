# quick A/B: tools/ab_quick.py for each variants/libcrn_<v>.so (outputs compared with the first variant's)
mkdir -p gpurun_out
TAG=${1:-abq}
shift
first=""
for v in "$@"; do
  [ -z "$first" ] && first=$v
  for r in 1 2; do
    CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_$v.so timeout 150 python tools/ab_quick.py --tag $v \
      --save /tmp/abq_$v.pt --ref /tmp/abq_$first.pt >> gpurun_out/${TAG}_summary.txt 2>> gpurun_out/${TAG}_err.txt
  done
done
