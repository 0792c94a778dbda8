"""Host->device copy bandwidth from pinned memory: one stream vs the same bytes split
across several streams (copy engines). Used to read the e2e line: e2e ~ max(epoch,
feature bytes / H2D rate)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


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
    print(json.dumps(probe()))
