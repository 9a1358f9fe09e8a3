"""Rank-count invariance on the GPU ("per-CB outputs are
identical for G in {1, 2, 4, 8}"): bench.py's real N-rank code
path is launched under torchrun with 1, 2 and 4 ranks sharing cuda:0 (gloo for
the host collectives; the ranks never wait on each other's kernels, so this is
a functional run, not a measurement), each rank decoding its cell shard; the
per-cell output digests of the strong split (cfg4's cells 0..7 over N ranks)
and of the weak batches (cells r*8..r*8+7 on rank r) must agree across N and
with the oracle's decode of the same cells."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_1905_01141_b200 import build as crn_build
from paper_1905_01141_b200 import shard
from paper_1905_01141_b200 import workload as wlmod
from tests._gpu import run_oracle
from tests._inputs import oracle_batch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CELLS = 8


def _run(n, out, port):
    env = dict(os.environ, CRN_BENCH_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
           "--gpus", str(n), "--steps", "1", "--warmup", "3", "--cells", str(CELLS), "--no-latency",
           "--no-pool", "--no-e2e", "--no-cpu-baseline", "--dist-backend", "gloo", "--digest-out", out]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    with open(out) as f:
        return line, json.load(f)


def _oracle_cell_digests(cells):
    """The oracle's decode of the same cells (inputs from the oracle's CRC and
    encoder), packed LSB-first into words like the decoder's out_bits."""
    wl = wlmod.make_workload(4, seed=0, cells=cells, device="cuda")
    b = oracle_batch(wl)
    idx = np.arange(b.n_cb)
    r = run_oracle(b, idx, 8, False)
    words = np.zeros(b.n_words, np.uint32)
    for i in idx:
        k = int(b.desc["K"][i])
        bits = r["bits"][r["bo"][i]:r["bo"][i] + k]
        w = np.packbits(np.r_[bits, np.zeros((-k) % 32, np.uint8)], bitorder="little").view(np.uint32)
        words[b.desc["bit_off"][i]:b.desc["bit_off"][i] + w.size] = w
    return shard.cell_digests(b.desc, b.cb_cell, words, r["crc_ok"])


def test_outputs_do_not_depend_on_rank_count(tmp_path, orc):
    crn_build.build()
    assert torch.cuda.is_available()
    res = {}
    for n in (1, 2, 4):
        line, dg = _run(n, str(tmp_path / f"d{n}.json"), 29400 + 13 * n + os.getpid() % 300)
        assert line["n_gpus"] == n and len(line["digests"]["per_rank"]) == n
        assert "functional_check_only" in line or n == 1
        res[n] = (line, {int(k): v for k, v in dg["strong"].items()}, {int(k): v for k, v in dg["weak"].items()})
    strong1 = res[1][1]
    assert sorted(strong1) == list(range(CELLS))
    for n in (2, 4):
        line, strong, weak = res[n]
        assert strong == strong1, f"strong split over {n} ranks decoded some cell differently"
        assert line["strong"]["cells_sha256"] == res[1][0]["strong"]["cells_sha256"]
        assert sorted(weak) == list(range(n * CELLS))
        for c in range(n * CELLS):                         # every weak cell equals its strong/N=1 decode
            if c in strong1:
                assert weak[c] == strong1[c]
        for c in range(CELLS, n * CELLS):                   # cells first seen at N > 1 agree across N
            for m in (2, 4):
                if m != n and c in res[m][2]:
                    assert res[m][2][c] == weak[c]
    assert _oracle_cell_digests(list(range(CELLS))) == strong1
