"""Critical-path analysis of the asynchronous GC run (DPC_TRACE=1): per JP
level, when its last vertex was colored; per-degree latency of the links."""
import os
import sys
import numpy as np
os.environ["DPC_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1606_08150_b200 as dpc  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
order_name = sys.argv[2] if len(sys.argv) > 2 else "canonical"  # the library default since round 2
ctx = dpc.Context(0)
g = dpc.gen_rmat(scale, 16, seed=1, weights=False, symmetric=True)
dg = dpc.DeviceGraph(ctx, g)
cfg = dpc.launch_cfg("color", "grid", gc_order=order_name)
dg.color(1, "grid", cfg=cfg)
ctx.flush_l2()
dg.color(1, "grid", cfg=cfg, metrics=False)
n = g.n
allt = dg.trace(3 * n).astype(np.int64)
ts, tq, td = allt[:n].copy(), allt[n:2 * n].copy(), allt[2 * n:].copy()
t0 = ts.min()
ts -= t0
tq -= t0
td -= t0
rp = g.rowptr
deg = np.diff(rp)


def mix64(z):
    z = (z + np.uint64(0x9E3779B97F4A7C15))
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


with np.errstate(over="ignore"):
    pr = mix64(np.arange(n, dtype=np.uint64) ^ np.uint64(1))
if order_name == "canonical":
    rank = np.arange(n, dtype=np.int64)  # node 0 first
else:
    order = np.lexsort((np.arange(n), pr))[::-1]
    rank = np.empty(n, np.int64)
    rank[order] = np.arange(n)
# level + the predecessor that colored last (critical predecessor)
src = np.repeat(np.arange(n), deg)
col = g.col.astype(np.int64)
hi = (rank[col] < rank[src]) & (col != src)
lev = np.zeros(n, np.int64)
# process in priority order (vectorised per vertex is slow in python: use the timestamps instead)
print("total span us", ts.max() / 1e3)
# per-vertex wait: ts[v] - max(ts[u] for higher u)
last_hi = np.full(n, -1, np.int64)
np.maximum.at(last_hi, src[hi], ts[col[hi]])
gap = np.where(last_hi >= 0, ts - last_hi, ts)
for lo, hi_ in [(0, 8), (8, 32), (32, 128), (128, 512), (512, 4096), (4096, 1 << 30)]:
    m = (deg >= lo) & (deg < hi_) & (last_hi >= 0)
    if m.any():
        print(f"deg [{lo},{hi_}): n={m.sum()} gap us median {np.median(gap[m]) / 1e3:.2f} p90 {np.percentile(gap[m], 90) / 1e3:.2f}")
# critical path: walk back from the last colored vertex
v = int(np.argmax(ts))
path = []
while True:
    path.append(v)
    nb = col[rp[v]:rp[v + 1]]
    hs = nb[(rank[nb] < rank[v]) & (nb != v)]
    if len(hs) == 0:
        break
    v = int(hs[np.argmax(ts[hs])])
path = path[::-1]
print("critical path length", len(path))
pp = np.array(path[1:])
prev = np.array(path[:-1])
print("  release->enqueue us median", np.median(tq[pp] - ts[prev]) / 1e3,
      " enqueue->dequeue", np.median(td[pp] - tq[pp]) / 1e3, " dequeue->color", np.median(ts[pp] - td[pp]) / 1e3)
m = (deg < 32) & (last_hi >= 0)
print("light vertices: release->enqueue", np.median(tq[m] - last_hi[m]) / 1e3, "enqueue->dequeue",
      np.median(td[m] - tq[m]) / 1e3, "dequeue->color", np.median(ts[m] - td[m]) / 1e3)
gaps = np.diff(ts[path])
print("path gap us: median", np.median(gaps) / 1e3, "mean", gaps.mean() / 1e3, "p90", np.percentile(gaps, 90) / 1e3)
pd = deg[path[1:]]
for lo, hi_ in [(0, 32), (32, 128), (128, 512), (512, 4096), (4096, 1 << 30)]:
    m = (pd >= lo) & (pd < hi_)
    if m.any():
        print(f"  path links into deg [{lo},{hi_}): {m.sum()} total {gaps[m].sum() / 1e3:.0f} us mean {gaps[m].mean() / 1e3:.2f}")
