"""Host link bandwidth of this box (pinned memory): H2D alone, D2H alone, both directions at once; chunked."""
import json
import time

import torch

n = 1 << 27  # 1 GiB of fp64
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.randn(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


def both_chunked(chunks=32):
    c = n // chunks
    for i in range(chunks):
        with torch.cuda.stream(s1):
            d_in[i * c:(i + 1) * c].copy_(h_in[i * c:(i + 1) * c], non_blocking=True)
        with torch.cuda.stream(s2):
            h_out[i * c:(i + 1) * c].copy_(d_out[i * c:(i + 1) * c], non_blocking=True)


B = 8 * n / 1e9
res["h2d_GBs"] = B / timed(h2d)
res["d2h_GBs"] = B / timed(d2h)
t = timed(both)
res["bidir_each_GBs"] = B / t
res["bidir_chunked_each_GBs"] = B / timed(both_chunked)
print(json.dumps(res))
