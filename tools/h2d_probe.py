"""Host<->device copy paths for the fp64 C2 latent (37.7 MB): pageable
cudaMemcpy, cudaHostRegister + copy, pinned staging. Probe, not a bench."""
import ctypes
import time

import numpy as np
import torch

n = 4096 * 1152
x = np.random.rand(n)
out = np.empty_like(x)
d = torch.empty(n, dtype=torch.float64, device="cuda")
cudart = ctypes.CDLL("libcudart.so.12") if False else None
torch.cuda.synchronize()


def t(f, reps=5):
    f()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        f()
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    return 1e3 * min(ts)


xt = torch.from_numpy(x)
ot = torch.from_numpy(out)
print("pageable H2D ms", t(lambda: d.copy_(xt)))
print("pageable D2H ms", t(lambda: ot.copy_(d)))
pin = torch.empty(n, dtype=torch.float64).pin_memory()
print("pinned H2D ms", t(lambda: d.copy_(pin, non_blocking=True)))
print("pinned D2H ms", t(lambda: pin.copy_(d, non_blocking=True)))
print("numpy->pinned memcpy ms", t(lambda: pin.numpy().__setitem__(slice(None), x)))
cr = torch.cuda.cudart()


def reg_copy():
    cr.cudaHostRegister(x.ctypes.data, x.nbytes, 0)
    d.copy_(xt, non_blocking=True)
    torch.cuda.synchronize()
    cr.cudaHostUnregister(x.ctypes.data)


print("register+H2D+unregister ms", t(reg_copy))
fresh = lambda: np.empty_like(x)
print("np.empty_like + D2H (page faults) ms", t(lambda: torch.from_numpy(fresh()).copy_(d)))
