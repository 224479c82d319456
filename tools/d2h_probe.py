import torch, time
n = 6_178_276_440 // 4
d = torch.empty(n, dtype=torch.int32, device="cuda")
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
for k in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(k)]
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        step = (n + k - 1) // k
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                h[i*step:(i+1)*step].copy_(d[i*step:(i+1)*step], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(f"D2H {k} streams: {dt*1e3:.1f} ms, {n*4/dt/1e9:.1f} GB/s", flush=True)
x = torch.empty(368_676_984 // 4, dtype=torch.int32, pin_memory=True)
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter(); y = x.to("cuda", non_blocking=True); torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"H2D 368MB: {dt*1e3:.1f} ms {x.numel()*4/dt/1e9:.1f} GB/s")
