#!/usr/bin/env python
"""Diagnostics: host link bandwidth with pinned buffers of the e2e step's size (2 x 57.5 MB
each way): H2D alone, D2H alone, both directions at once (two streams). Not a bench line."""
import json

import torch

n = 7189057 * 2
h_in = torch.empty(n, dtype=torch.float64).pin_memory()
h_out = torch.empty(n, dtype=torch.float64).pin_memory()
d_in = torch.empty(n, dtype=torch.float64, device="cuda")
d_out = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
B = n * 8


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"bytes_each_way": B, "h2d_ms": t1, "h2d_gbs": B / t1 / 1e6, "d2h_ms": t2, "d2h_gbs": B / t2 / 1e6,
                  "duplex_ms": t3, "duplex_gbs_each_way": B / t3 / 1e6}))
