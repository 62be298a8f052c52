import torch, time
n = 768 * 2**20 // 8
d = torch.randn(n, dtype=torch.float64, device="cuda")
h = torch.empty(n, dtype=torch.float64).pin_memory()
for chunks in (1, 3, 6, 12):
    s = [torch.cuda.Stream() for _ in range(2)]
    torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        t0 = time.perf_counter()
        cs = n // chunks
        for i in range(chunks):
            st = s[i % 2]
            with torch.cuda.stream(st):
                h[i*cs:(i+1)*cs].copy_(d[i*cs:(i+1)*cs], non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    print(f"chunks {chunks}: {n*8/best/1e9:.1f} GB/s")
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
torch.cuda.synchronize(); t0=time.perf_counter(); h2.copy_(d, non_blocking=True); torch.cuda.synchronize(); print("single", n*8/(time.perf_counter()-t0)/1e9)
