import sys, os, time, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2407_09621_b200 as sf
from paper_2407_09621_b200 import discretization as dz
hier = sf.build_hierarchy(7, 7, max_dofs=2**34, min_level=7)
D = hier.n_dofs(7)
u = torch.randn(D, dtype=torch.float64).pin_memory()
v = torch.empty_like(u).pin_memory()
out = {}
for sc in (2, 4, 2, 4, 2, 4):
    dz._stream_vmult(hier, 7, u, v, sf.PrecisionMode.FP64, slab_cells=sc)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3): dz._stream_vmult(hier, 7, u, v, sf.PrecisionMode.FP64, slab_cells=sc)
    torch.cuda.synchronize()
    out.setdefault(f"slab{sc}", []).append(round(3 * D / (time.perf_counter() - t) / 1e9, 3))
ref = torch.empty(D, dtype=torch.float64, device="cuda")
dz.vmult_device(hier, 7, u.cuda(), ref, sf.PrecisionMode.FP64)
out["max_abs_diff"] = float((v.cuda() - ref).abs().max())
print(json.dumps(out))
