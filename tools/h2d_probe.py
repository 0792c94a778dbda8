"""Host->device copy bandwidth from pinned memory: one stream vs the same bytes split
across several streams (copy engines). Used to read the e2e line: e2e ~ max(epoch,
feature bytes / H2D rate)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _load(kind: str, dev):
    """A concurrent load on a side stream: 'l2' gathers random 256-byte rows of a 60 MB
    (L2-resident) matrix like the aggregation; 'hbm' streams a 4 GB device copy."""
    if kind == "l2":
        src = torch.randn(233_000, 64, device=dev)
        idx = torch.randint(0, 233_000, (8_000_000,), device=dev)
        return lambda: torch.index_select(src, 0, idx)
    a = torch.empty(1 << 30, dtype=torch.float32, device=dev)
    b = torch.empty_like(a)
    return lambda: b.copy_(a)


def probe_under_load(kind: str, nbytes: int = 562 << 20, reps: int = 3):
    dev = torch.device("cuda:0")
    n = nbytes // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    d = torch.empty(n, dtype=torch.float32, device=dev)
    work = _load(kind, dev)
    ls = torch.cuda.Stream(device=dev)
    cs = torch.cuda.Stream(device=dev)
    best = 0.0
    for _ in range(reps):
        torch.cuda.synchronize()
        with torch.cuda.stream(ls):
            for _ in range(40):
                work()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(cs):
            e0.record(cs)
            d.copy_(h, non_blocking=True)
            e1.record(cs)
        torch.cuda.synchronize()
        best = max(best, nbytes / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    return round(best, 1)


def probe(nbytes: int = 562 << 20, reps: int = 5):
    dev = torch.device("cuda:0")
    n = nbytes // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float32, device=dev)
    out = {}
    for k in (1, 2, 4):
        streams = [torch.cuda.Stream(device=dev) for _ in range(k)]
        chunk = (n + k - 1) // k
        best = 0.0
        for _ in range(reps):
            torch.cuda.synchronize()
            s0 = torch.cuda.Event(enable_timing=True)
            s1 = torch.cuda.Event(enable_timing=True)
            cur = torch.cuda.current_stream()
            s0.record(cur)
            for i, s in enumerate(streams):
                s.wait_stream(cur)
                with torch.cuda.stream(s):
                    d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
            for s in streams:
                cur.wait_stream(s)
            s1.record(cur)
            torch.cuda.synchronize()
            best = max(best, nbytes / (s0.elapsed_time(s1) * 1e-3) / 1e9)
        out[f"streams_{k}_gbs"] = round(best, 1)
    return out


if __name__ == "__main__":
    r = probe()
    if "--load" in sys.argv:
        r["under_l2_gather_gbs"] = probe_under_load("l2")
        r["under_hbm_stream_gbs"] = probe_under_load("hbm")
    print(json.dumps(r))
