"""PCIe copy bandwidth on this box (dev aid): pinned H2D / D2H of 134 MB on
1, 2 and 4 streams."""
import time
import torch

nbytes = 134 << 20
dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
for direction in ("d2h", "h2d"):
    for ns in (1, 2, 4):
        streams = [torch.cuda.Stream() for _ in range(ns)]
        chunk = nbytes // ns
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    if direction == "d2h":
                        host[i * chunk:(i + 1) * chunk].copy_(dev[i * chunk:(i + 1) * chunk], non_blocking=True)
                    else:
                        dev[i * chunk:(i + 1) * chunk].copy_(host[i * chunk:(i + 1) * chunk], non_blocking=True)
            torch.cuda.synchronize()
            best = min(best, time.perf_counter() - t0)
        print(f"{direction} {ns} streams: {nbytes / best / 1e9:.1f} GB/s ({best * 1e3:.2f} ms)")
