# round-2 baseline: ncu launch list + full capture of the decode kernel, phase profiles (cfg4 / cfg3 / cfg5)
mkdir -p gpurun_out
TAG=${1:-r2e}
bash tools/jobs/prof.sh $TAG
for c in "64 4" "100 3" "20 5"; do
  set -- $c
  CRN_LIB=$PWD/paper_1905_01141_b200/libcrn_prof.so timeout 300 python tools/phase_prof.py $1 $2 > gpurun_out/${TAG}_phase_cfg$2.json 2>&1
done
