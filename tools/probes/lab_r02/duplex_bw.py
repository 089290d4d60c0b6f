"""Concurrent H2D + D2H pinned copies (two streams) vs each alone: the
aggregate PCIe throughput the pipelined e2e path can reach on this box."""
import torch

n = 4 << 20  # 4 MB per direction, like one config-2 vector
for mb in (4, 64):
    nb = mb << 20
    ha = torch.empty(nb, dtype=torch.uint8).pin_memory()
    hb = torch.empty(nb, dtype=torch.uint8).pin_memory()
    da = torch.empty(nb, dtype=torch.uint8, device="cuda")
    db = torch.empty(nb, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for mode in ("h2d", "d2h", "both"):
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            s1.wait_event(e0)
            s2.wait_event(e0)
            if mode in ("h2d", "both"):
                with torch.cuda.stream(s1):
                    da.copy_(ha, non_blocking=True)
            if mode in ("d2h", "both"):
                with torch.cuda.stream(s2):
                    hb.copy_(db, non_blocking=True)
            torch.cuda.current_stream().wait_stream(s1)
            torch.cuda.current_stream().wait_stream(s2)
            e1.record()
            torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1))
        moved = nb * (2 if mode == "both" else 1)
        print(f"{mb:3d} MB {mode:4s}: {best * 1e3:7.1f} us  {moved / (best * 1e-3) / 1e9:6.1f} GB/s aggregate", flush=True)
