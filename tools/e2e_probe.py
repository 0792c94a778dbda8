"""Probe of the end-to-end step pieces on the Reddit-shape workload: the pinned H2D
of one feature block alone, the epoch alone (native C-ABI trainer vs the
torch-orchestrated trainer, CUDA-graph replays), and the pipelined staged loop."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import paper_2311_06837_b200 as G
    from paper_2311_06837_b200.native import NativeTrainer
    from paper_2311_06837_b200.train import FullGraphTrainer, ModelConfig

    d = torch.device("cuda", 0)
    g = G.gen_random_graph(232965, 491.99, 11)
    cfg = ModelConfig("sage", [602, 64, 64, 41], lr=0.1)
    out = {}
    nt = NativeTrainer(g, cfg)
    s = nt.stream()
    for _ in range(4):
        nt.train_epoch(sync_loss=False)
    torch.cuda.synchronize()

    def timed(fn, reps, stream=None):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(reps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    out["native_epoch_ms"] = timed(lambda: nt.train_epoch(sync_loss=False), 20, s)
    ft = FullGraphTrainer(g, cfg)
    ft.capture(warmup=2)
    out["torch_epoch_ms"] = timed(ft.replay, 20)
    out["native_epoch_ms_again"] = timed(lambda: nt.train_epoch(sync_loss=False), 20, s)
    xh = torch.empty((nt.nloc, 602), dtype=torch.float32).pin_memory()
    xh.uniform_(-0.5, 0.5)
    lh = torch.zeros(nt.nloc, dtype=torch.int32).pin_memory()
    xd = torch.empty((nt.nloc, 602), dtype=torch.float32, device=d)
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        out["torch_h2d_ms"] = timed(lambda: xd.copy_(xh, non_blocking=True), 5, cs)
    t = time.perf_counter()
    for _ in range(5):
        nt.stage_inputs(None, x_ptr=xh.data_ptr(), labels_ptr=lh.data_ptr())
        nt.step_staged(sync_loss=True)
    out["staged_serial_ms"] = (time.perf_counter() - t) / 5 * 1e3
    t = time.perf_counter()
    nt.stage_inputs(None, x_ptr=xh.data_ptr(), labels_ptr=lh.data_ptr())
    for i in range(10):
        if i + 1 < 10:
            nt.stage_inputs(None, x_ptr=xh.data_ptr(), labels_ptr=lh.data_ptr())
        nt.step_staged(sync_loss=True)
    out["staged_pipelined_ms"] = (time.perf_counter() - t) / 10 * 1e3
    print(json.dumps(out))


if __name__ == "__main__":
    main()
