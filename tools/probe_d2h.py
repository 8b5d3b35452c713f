"""Pinned device->host copy bandwidth with 1, 2 and 4 concurrent streams
(what bounds the e2e ids stream): python tools/probe_d2h.py"""
import torch
torch.cuda.set_device(0)
nbytes = 200 << 20
src = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
dst = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = nbytes // ns
    for it in range(2):
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for k, s in enumerate(streams):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                dst[k * chunk:(k + 1) * chunk].copy_(src[k * chunk:(k + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"streams {ns}: {nbytes / ms / 1e6:.1f} GB/s ({ms:.2f} ms for 200 MiB)", flush=True)
