"""Host->device copy bandwidth from pinned memory with 1..4 concurrent streams
(what the e2e leg of bench.py is bounded by)."""
import json
import torch

N = 1 << 30  # bytes per copy
src = torch.empty(4 * N // 2, dtype=torch.bfloat16).pin_memory()
dst = torch.empty(4 * N // 2, dtype=torch.bfloat16, device="cuda")
for ns in (1, 2, 3, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = src.numel() // ns
    for rep in range(2):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                dst[i * chunk:(i + 1) * chunk].copy_(src[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"streams": ns, "GB": 4 * N / 1e9, "ms": ms, "GBps": 4 * N / ms / 1e6}))
# d2h for reference
h = torch.empty(N // 2, dtype=torch.bfloat16).pin_memory()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); h.copy_(dst[:N // 2], non_blocking=True); e1.record(); torch.cuda.synchronize()
print(json.dumps({"d2h_GBps": N / e0.elapsed_time(e1) / 1e6}))
