"""Regenerate the golden fixtures from the REFERENCE ITSELF (oracle/_ref,
built from /root/reference by `make -C oracle ref`).

    python tests/golden/make_golden.py

Fixtures (committed):
  cref.npz    reference_execute.cfg (proj/configs/reference_execute.cfg:4-17):
              L=4 hs=32 heads=4 p=64 S=20 N=M=4 W=1 eta=0.1 seed=0
  c1_s4.npz   BASELINE config 1 (tiny): L=4 hs=128 heads=4 p=256 N=2 M=4 W=1, S=4
  c1_s5.npz   same with S=5 (the "4 steps + 1 warmup" reading)
Each holds the PipeFusion final latent (Threads backend, the CLI default), the
serial_reference final latent, the StalenessStats and the divergence.
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.loader import Reference  # noqa: E402

CASES = {
    "cref": dict(seed=0, L=4, hs=32, heads=4, p=64, S=20, N=4, M=4, W=1, eta=0.1),
    "c1_s4": dict(seed=0, L=4, hs=128, heads=4, p=256, S=4, N=2, M=4, W=1, eta=0.1),
    "c1_s5": dict(seed=0, L=4, hs=128, heads=4, p=256, S=5, N=2, M=4, W=1, eta=0.1),
}


def make(name, c, ref):
    m = ref.build_toy_model(c["seed"], c["L"], c["hs"], c["heads"], 4.0)
    x0 = ref.make_initial_latent(c["seed"], c["p"], c["hs"])
    serial = m.serial_reference(x0, c["S"], c["eta"])
    pf, (fresh, stale, ff) = m.run_pipefusion(x0, c["S"], c["N"], c["M"], c["W"], c["eta"])
    div = ref.divergence(pf, serial)
    np.savez(Path(__file__).parent / f"{name}.npz", x_pipefusion=pf, x_serial=serial,
             fresh=fresh, stale=stale, fresh_fraction=np.asarray(ff), divergence=div,
             config=np.array(repr(c)))
    print(name, "divergence", repr(div), "fresh/stale", fresh, stale)


if __name__ == "__main__":
    ref = Reference()
    for name, c in CASES.items():
        make(name, c, ref)
