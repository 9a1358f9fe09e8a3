# parity + short bench, then the ncu launch list + one full capture
TAG=${1:-q}
bash tools/jobs/quick.sh $TAG
grep -q "pytest rc=0" gpurun_out/${TAG}_rc.txt && bash tools/jobs/prof.sh $TAG
