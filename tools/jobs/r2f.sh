mkdir -p gpurun_out
TAG=${1:-r2f}
for c in "64 4" "100 3" "20 5"; do
  set -- $c
  CRN_LIB=$PWD/paper_1905_01141_b200/libcrn_prof.so timeout 300 python tools/phase_prof.py $1 $2 > gpurun_out/${TAG}_phase_cfg$2.json 2>&1
done
bash tools/jobs/abq.sh ${TAG}_ab base qoff base qoff
