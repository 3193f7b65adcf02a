"""Host-side breakdown of one e2e step (upload / run / download / whole call)
on config 2; diagnostic only (not a bench number)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
from paper_1711_08475_b200 import GpuFingerprintedDictionary, QueryOptions  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
c, blob, offs, qblob, qoffs, scheme, metric, first, n = bench.workload(cfg, 0, 0, 1)
qb, qo = bench.pinned_copy(qblob), bench.pinned_copy(qoffs)
opt = QueryOptions(metric, 1, True, True)
d = GpuFingerprintedDictionary((blob, offs), scheme, devices=(0,), keep_words=False)
b = d.batch()
T = {"upload": [], "run": [], "download": [], "query_batch": [], "run_ms(dev)": []}
for it in range(30):
    t0 = time.perf_counter(); b.upload(qb, qo); t1 = time.perf_counter()
    b.run(opt, want_stats=True); t2 = time.perf_counter()
    b.download(); t3 = time.perf_counter()
    d.query_batch((qb, qo), opt, per_query_stats=True); t4 = time.perf_counter()
    if it >= 5:
        T["upload"].append(t1 - t0); T["run"].append(t2 - t1); T["download"].append(t3 - t2)
        T["query_batch"].append(t4 - t3); T["run_ms(dev)"].append(b.timing()["run_ms"] / 1e3)
for k, v in T.items():
    print(f"{k:14s} median {1e3 * np.median(v):8.3f} ms")
