# smoke + ubench + gpu tests + bench + ncu launch list + one full capture of the decode kernel
set -x
mkdir -p gpurun_out
TAG=${1:-cur}
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
nproc > gpurun_out/nproc.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 300 python tools/ubench.py > gpurun_out/${TAG}_ubench.json 2>&1; echo "ubench rc=$?" >> gpurun_out/rc.txt
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/rc.txt
bash tools/jobs/prof.sh ${TAG}
