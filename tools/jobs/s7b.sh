# session 6: one full ncu capture of the TB conditioning kernel on cfg3's 1,000 TBs
mkdir -p gpurun_out
TAG=${1:-s7b}
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tbseg_kernel -s 3 -c 1 -o gpurun_out/${TAG}_tbseg \
  python -c "import bench; bench.run_dl_encode_tb(reps=1)" > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/${TAG}_rc.txt
