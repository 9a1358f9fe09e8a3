mkdir -p gpurun_out
TAG=r2l
bash tools/jobs/abq.sh ${TAG}_ab hd1 pre bulkp hd1 pre bulkp
for v in prof_pre prof_bulkp; do
for c in "64 4" "100 3"; do
  set -- $c
  CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_$v.so timeout 120 python tools/phase_prof.py $1 $2 > gpurun_out/${TAG}_${v}_cfg$2.json 2>&1
done
done
