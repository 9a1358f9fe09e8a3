# rate matching rewrite: parity tests + DL kernel times, old vs new
mkdir -p gpurun_out
TAG=${1:-s4g}
timeout 600 python -m pytest tests -m gpu -q -k "rate or packed or encoder" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_summary.txt
for v in rmbase rmnew rmbase rmnew; do
  echo -n "$v " >> gpurun_out/${TAG}_summary.txt
  CRN_LIB=$PWD/paper_1905_01141_b200/variants/libcrn_$v.so timeout 300 python tools/dl_time.py 256 >> gpurun_out/${TAG}_summary.txt 2>> gpurun_out/${TAG}_err.txt
done
