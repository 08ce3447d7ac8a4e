import torch, time
N = 6_400_000_000 // 4
h = torch.empty(N, dtype=torch.int32, pin_memory=True)
d = torch.empty(N, dtype=torch.int32, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        step = (N + ns - 1) // ns
        for k, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[k * step:(k + 1) * step].copy_(h[k * step:(k + 1) * step], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
    print(f"{ns} streams: {dt*1e3:.1f} ms  {N*4/dt/1e9:.1f} GB/s", flush=True)
# chunked single stream 16 pieces
torch.cuda.synchronize(); t = time.perf_counter()
step = N // 16
for k in range(16):
    d[k*step:(k+1)*step].copy_(h[k*step:(k+1)*step], non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"16 pieces 1 stream: {dt*1e3:.1f} ms  {N*4/dt/1e9:.1f} GB/s")
