"""PCIe probe: H2D GB/s with 1/2/4 concurrent copy streams, alone and beside a D2H copy."""
import torch, time
n = 4 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
dh = torch.empty(n // 4, dtype=torch.uint8).pin_memory()
dd = torch.empty(n // 4, dtype=torch.uint8, device="cuda")
def run(k, with_d2h=False):
    ss = [torch.cuda.Stream() for _ in range(k)]
    s2 = torch.cuda.Stream()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for rep in range(3):
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * n // k:(i + 1) * n // k].copy_(h[i * n // k:(i + 1) * n // k], non_blocking=True)
        if with_d2h:
            with torch.cuda.stream(s2):
                dh.copy_(dd, non_blocking=True)
    torch.cuda.synchronize()
    return 3 * n / (time.perf_counter() - t) / 1e9
for k in (1, 2, 4):
    print("h2d streams", k, round(run(k), 1), "GB/s;  with concurrent d2h", round(run(k, True), 1))
