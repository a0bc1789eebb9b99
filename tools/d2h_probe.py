"""D2H bandwidth of a 4 GiB device buffer into pinned memory: one copy vs row chunks on
two copy streams (the MatrixBuffer.download strategy)."""
import torch, time
n = 4 << 30  # 4 GiB
src = torch.empty(n, dtype=torch.uint8, device='cuda')
dst = torch.empty(n, dtype=torch.uint8, pin_memory=True)
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    ch = n // ns
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for k, s in enumerate(streams):
            with torch.cuda.stream(s):
                dst[k*ch:(k+1)*ch].copy_(src[k*ch:(k+1)*ch], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(ns, 'streams', n/dt/1e9, 'GB/s', flush=True)
# h2d
for ns in (1, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    ch = n // ns
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        for k, s in enumerate(streams):
            with torch.cuda.stream(s):
                src[k*ch:(k+1)*ch].copy_(dst[k*ch:(k+1)*ch], non_blocking=True)
        torch.cuda.synchronize(); dt = time.perf_counter() - t
    print('h2d', ns, 'streams', n/dt/1e9, 'GB/s', flush=True)
