import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2308_00106_b200.permute import pcg64_swap_partners_device
torch.zeros(1, device='cuda')
for n in (50_000_000, 8_000_000):
    for rep in range(3):
        torch.cuda.synchronize(); t = time.perf_counter()
        pcg64_swap_partners_device(np.random.PCG64(rep), n)
        torch.cuda.synchronize(); print(n, f"{time.perf_counter() - t:.4f} s", flush=True)

from concurrent.futures import ThreadPoolExecutor

n = 50_000_000
for rep in range(3):
    torch.cuda.synchronize()
    t = time.perf_counter()
    with ThreadPoolExecutor(max_workers=2) as ex:
        list(ex.map(lambda s: pcg64_swap_partners_device(np.random.PCG64(s), n), [1, 2]))
    torch.cuda.synchronize()
    print(f"two axes concurrently: {time.perf_counter() - t:.4f} s", flush=True)
