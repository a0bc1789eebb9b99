"""Device -> host copy paths for API results (MatrixBuffer.data, statistics): pageable
.cpu(), a pinned block of the caching host allocator, and a fresh numpy array."""
import time, torch, json
for nbytes in (8 << 20, 800 << 20, 4 << 30):
    src = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda").fill_(1.0)
    torch.cuda.synchronize()
    for rep in range(2):
        t0 = time.perf_counter(); a = src.cpu().numpy(); t1 = time.perf_counter()
        p = torch.empty(src.shape, dtype=src.dtype, pin_memory=True); t2 = time.perf_counter()
        p.copy_(src); b = p.numpy(); t3 = time.perf_counter()
        # fresh numpy destination registered on the fly
        import numpy as np
        h = np.empty(src.shape, np.float64); t4 = time.perf_counter()
        torch.from_numpy(h).copy_(src); t5 = time.perf_counter()
        print(json.dumps({"MB": nbytes >> 20, "rep": rep, "pageable_cpu_ms": round((t1-t0)*1e3, 2),
                          "pinned_alloc_ms": round((t2-t1)*1e3, 2), "pinned_copy_ms": round((t3-t2)*1e3, 2),
                          "np_empty_copy_ms": round((t5-t4)*1e3, 2)}), flush=True)
        del a, b, p, h
    del src
