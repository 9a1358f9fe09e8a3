# lone-warp latency study: ncu source captures of a cfg5 TTI and of cfg1, phase profiles of cfg1 / cfg5 / cfg3
mkdir -p gpurun_out
TAG=${1:-s4b}
for c in 5 1; do
  timeout 300 python tools/small_decode.py $c > gpurun_out/${TAG}_plain$c.log 2>&1 && \
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 \
      -o gpurun_out/${TAG}_cfg$c python tools/small_decode.py $c > gpurun_out/${TAG}_ncu$c.log 2>&1
  echo "ncu cfg$c rc=$?" >> gpurun_out/${TAG}_rc.txt
done
for c in "20 5" "32 1" "100 3"; do
  set -- $c
  CRN_LIB=$PWD/paper_1905_01141_b200/libcrn_prof.so timeout 300 python tools/phase_prof.py $1 $2 > gpurun_out/${TAG}_phase_cfg$2.json 2>&1
done
