# phase profile of the latency kernels (cfg1 spread, cfg5 one TTI) and of cfg2
mkdir -p gpurun_out
TAG=${1:-s4i}
for c in "32 1" "20 5" "1 2"; do
  set -- $c
  CRN_LIB=$PWD/paper_1905_01141_b200/libcrn_prof.so timeout 300 python tools/phase_prof.py $1 $2 > gpurun_out/${TAG}_phase_cfg$2.json 2>&1
done
