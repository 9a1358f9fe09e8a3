# round-2 first evidence run: smoke, full pytest -m gpu, default bench line, phase profiles (cfg3 ET / cfg4)
mkdir -p gpurun_out
TAG=${1:-r2b}
nvidia-smi > gpurun_out/${TAG}_nvsmi.txt 2>&1; nproc >> gpurun_out/${TAG}_nvsmi.txt
timeout 300 python __graft_entry__.py smoke > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/${TAG}_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 900 python bench.py > gpurun_out/${TAG}_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/${TAG}_rc.txt
CRN_LIB=paper_1905_01141_b200/libcrn_prof.so timeout 300 python tools/phase_prof.py 100 3 > gpurun_out/${TAG}_phase_cfg3.json 2>&1; echo "prof3 rc=$?" >> gpurun_out/${TAG}_rc.txt
CRN_LIB=paper_1905_01141_b200/libcrn_prof.so timeout 300 python tools/phase_prof.py 64 4 > gpurun_out/${TAG}_phase_cfg4.json 2>&1; echo "prof4 rc=$?" >> gpurun_out/${TAG}_rc.txt
