import time, torch
nb = 134 << 20
d1 = torch.empty(nb, dtype=torch.uint8, device="cuda"); d2 = torch.empty(nb // 2, dtype=torch.uint8, device="cuda")
h1 = torch.empty(nb, dtype=torch.uint8).pin_memory(); h2 = torch.empty(nb // 2, dtype=torch.uint8).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); t = time.perf_counter() - t0
print(f"bidirectional: 134 MB H2D + 67 MB D2H concurrently: {t*1e3:.2f} ms")
