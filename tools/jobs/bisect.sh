# usage: bash tools/jobs/bisect.sh TAG v1 v2 ... : smoke with each variants/libcrn_<v>.so
mkdir -p gpurun_out
TAG=$1; shift
for v in "$@"; do
  CRN_LIB=paper_1905_01141_b200/variants/libcrn_$v.so timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_$v.log 2>&1
  echo "$v rc=$?" >> gpurun_out/${TAG}_rc.txt
done
