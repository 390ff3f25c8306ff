import torch, time
N = 3_200_000_000 // 8
h = torch.empty(N, dtype=torch.float64).pin_memory()
d = torch.empty(N, dtype=torch.float64, device="cuda")
d2 = torch.empty(N, dtype=torch.float64, device="cuda")
up, dn = torch.cuda.Stream(), torch.cuda.Stream()
def run(chunk_mb, same=True):
    ch = chunk_mb * (1 << 20) // 8
    n = (N + ch - 1) // ch
    evs = [torch.cuda.Event() for _ in range(n)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    for c in range(n):
        a = c * ch; b = min(N, a + ch)
        with torch.cuda.stream(dn):
            h[a:b].copy_(d[a:b], non_blocking=True); evs[c].record(dn)
    for c in range(n):
        a = c * ch; b = min(N, a + ch)
        with torch.cuda.stream(up):
            up.wait_event(evs[c]); d2[a:b].copy_(h[a:b], non_blocking=True)
    torch.cuda.synchronize()
    return (time.perf_counter() - t) * 1e3
def sep(chunk_mb):
    torch.cuda.synchronize(); t = time.perf_counter()
    with torch.cuda.stream(dn): h.copy_(d, non_blocking=True)
    torch.cuda.synchronize(); t1 = time.perf_counter()
    with torch.cuda.stream(up): d2.copy_(h, non_blocking=True)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    return (t1 - t) * 1e3, (t2 - t1) * 1e3
print("down alone, up alone ms", sep(0))
h2 = torch.empty(N, dtype=torch.float64).pin_memory()
torch.cuda.synchronize(); t = time.perf_counter()
with torch.cuda.stream(dn): h.copy_(d, non_blocking=True)
with torch.cuda.stream(up): d2.copy_(h2, non_blocking=True)
torch.cuda.synchronize(); print("duplex different buffers ms", (time.perf_counter() - t) * 1e3)
for mb in (16, 64, 256):
    run(mb); print("pipelined chunk", mb, "ms", run(mb))
