"""Host-side breakdown of the bench's e2e step (upload / run / download =
D2H wait + host assembly) on a config cell; diagnostic only (not a bench
number).  usage: python tools/e2e_breakdown.py [cfg] [cell]"""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1711_08475_b200 import GpuFingerprintedDictionary, QueryOptions  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
cell = int(sys.argv[2]) if len(sys.argv) > 2 else 0
HOLD = len(sys.argv) > 3 and sys.argv[3] == "hold"
held = None
w = bench.Workload(cfg, cell)
qb, qo = bench.pinned_copy(w.qblob), bench.pinned_copy(w.qoffs)
opt = QueryOptions(w.metric, 1, True, True)
d = GpuFingerprintedDictionary((w.blob, w.offs), w.scheme, devices=(0,), keep_words=False)
b = d.batch()
T = {k: [] for k in ("upload", "run", "download", "d2h_wait", "assemble", "run_ms(dev)")}
for it in range(8):
    t0 = time.perf_counter(); b.upload(qb, qo); t1 = time.perf_counter()
    b.run(opt, want_stats=True); t2 = time.perf_counter()
    out = b.download(); t3 = time.perf_counter()
    if HOLD:
        held = out  # like bench.py: the previous result stays alive during the next step
    del out
    if it >= 2:
        h = b.host_ms()
        T["upload"].append(t1 - t0); T["run"].append(t2 - t1); T["download"].append(t3 - t2)
        T["d2h_wait"].append(h["download_ms"] / 1e3); T["assemble"].append(h["assemble_ms"] / 1e3)
        T["run_ms(dev)"].append(b.timing()["run_ms"] / 1e3)
for k, v in T.items():
    print(f"{k:14s} median {1e3 * np.median(v):8.3f} ms")
