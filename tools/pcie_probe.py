"""Host-link probe: pinned H2D / D2H / concurrent bandwidth, and the streamed vmult at several slab sizes."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2407_09621_b200 as sf
from paper_2407_09621_b200 import discretization as dz

n = 1 << 28  # 2 GiB of f64
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def bw(fn, nbytes, reps=3):
    fn(); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps): fn()
    torch.cuda.synchronize()
    return nbytes * reps / (time.perf_counter() - t) / 1e9
out = {}
out["h2d_GBs"] = bw(lambda: d.copy_(h, non_blocking=True), 8 * n)
out["d2h_GBs"] = bw(lambda: h.copy_(d, non_blocking=True), 8 * n)
def both():
    with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
out["concurrent_total_GBs"] = bw(both, 16 * n)
del h, h2, d, d2
hier = sf.build_hierarchy(7, 7, max_dofs=2**34, min_level=7)
D = hier.n_dofs(7)
u = torch.randn(D, dtype=torch.float64).pin_memory()
v = torch.empty_like(u).pin_memory()
for sc in (2, 4, 8, 16, 32):
    dz._stream_vmult(hier, 7, u, v, sf.PrecisionMode.FP64, slab_cells=sc)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(2): dz._stream_vmult(hier, 7, u, v, sf.PrecisionMode.FP64, slab_cells=sc)
    torch.cuda.synchronize()
    out[f"stream_slab{sc}_gdofs"] = 2 * D / (time.perf_counter() - t) / 1e9
print(json.dumps(out))
