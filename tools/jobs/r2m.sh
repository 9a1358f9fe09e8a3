mkdir -p gpurun_out
TAG=r2m
bash tools/jobs/abq.sh ${TAG}_ab hd1 hdpf hd1 hdpf
for c in "64 4" "100 3"; do
  set -- $c
  CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_prof_hdpf.so timeout 120 python tools/phase_prof.py $1 $2 > gpurun_out/${TAG}_phase_cfg$2.json 2>&1
done
# is compute-sanitizer usable on this pool?
timeout 240 compute-sanitizer --tool memcheck --print-limit 20 python tools/small_decode.py 1 > gpurun_out/${TAG}_memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 300 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 python tools/small_decode.py 1 > gpurun_out/${TAG}_racecheck.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/${TAG}_rc.txt
