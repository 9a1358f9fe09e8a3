# phase profiles of profiling variants on cfg4: variants/libcrn_<v>.so (or the main libcrn_prof.so for "prof")
mkdir -p gpurun_out
TAG=${1:-pexp}
shift
for v in "$@"; do
  L=$PWD/paper_1905_01141_b200/variants/libcrn_$v.so
  [ "$v" = prof ] && L=$PWD/paper_1905_01141_b200/libcrn_prof.so
  CRN_LIB=$L timeout 300 python tools/phase_prof.py 64 4 > gpurun_out/${TAG}_$v.json 2>&1
done
