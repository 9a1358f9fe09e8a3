mkdir -p gpurun_out
TAG=r2k
bash tools/jobs/abq.sh ${TAG}_ab hd1 bulk2 hd1 bulk2
for c in "64 4" "100 3"; do
  set -- $c
  CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_prof_bulk2.so timeout 120 python tools/phase_prof.py $1 $2 > gpurun_out/${TAG}_phase_cfg$2.json 2>&1
done
