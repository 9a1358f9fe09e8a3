# session 6: TB conditioning kernel (eight positions per thread in the pack and CB write stages): parity, per-call and kernel times
mkdir -p gpurun_out
TAG=${1:-s6b}
timeout 600 python -m pytest tests -m gpu -q -x -k "tb_build or encoder or dl_ or packed or batch" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 300 python - > gpurun_out/${TAG}_dl_tb.json 2>gpurun_out/${TAG}_dl_tb.err <<'P'
import json, torch, bench
print(json.dumps(bench.run_dl_encode_tb()))
P
echo "dl_tb rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tbseg --csv --log-file gpurun_out/${TAG}_tbseg_launches.csv \
  python -c "import bench; bench.run_dl_encode_tb(reps=1)" > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/${TAG}_rc.txt
