# session 6 (s6c, s6d): TB conditioning tables built once per device; default mempool release threshold raised at context init: DL per-call times again + host submit time of the TB conditioning call
mkdir -p gpurun_out
TAG=${1:-s6c}
timeout 600 python - > gpurun_out/${TAG}_dl.json 2>gpurun_out/${TAG}_dl.err <<'P'
import json, time, numpy as np, torch, bench
from paper_1905_01141_b200 import crn, workload as wlmod
print(json.dumps({"dl_encode_tb": bench.run_dl_encode_tb()}))
wl = wlmod.make_workload(3, seed=0, device="cuda")
tbs = np.asarray(wl.tbs, np.int64); pay = torch.cat(wl.payload)
off = np.concatenate([[0], np.cumsum(tbs)[:-1]]).astype(np.int64)
desc, info = crn.tb_build_cbs_batch(tbs, off, pay)
buf = torch.empty(int(desc["K"].sum()), dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream()
out = []
for _ in range(5):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(5): crn.tb_build_cbs_batch(tbs, off, pay, cb_bits=buf, max_cb=desc.size, stream=st)
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    out.append({"host_submit_us_per_call": (t1 - t) / 5 * 1e6, "wall_us_per_call": (t2 - t) / 5 * 1e6})
print(json.dumps({"tb_build_host": out}))
P
echo "dl rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_rc.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:tbseg --csv --log-file gpurun_out/${TAG}_tbseg_launches.csv \
  python -c "import bench; bench.run_dl_encode_tb(reps=1)" > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?" >> gpurun_out/${TAG}_rc.txt
