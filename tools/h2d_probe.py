import torch, time
n = 2 * 1024**3 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
h.fill_(1.0)
d = torch.empty(n, dtype=torch.float32, device="cuda")
torch.cuda.synchronize()
for nst in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(nst)]
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        ch = n // nst
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * ch:(i + 1) * ch].copy_(h[i * ch:(i + 1) * ch], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"{nst} stream(s): {n * 4 / dt / 1e9:.1f} GB/s")
torch.cuda.synchronize(); t0 = time.perf_counter()
x = h.to("cuda"); torch.cuda.synchronize(); print(f".to(cuda): {n*4/(time.perf_counter()-t0)/1e9:.1f} GB/s")
