"""End-to-end PipeFusion on the GPU vs the fp64 numpy restatement, on random
(non-reference) weights. The bit-exact reference-weight parity lives in
test_gpu_parity.py; this one isolates the executor from the RNG restatement.
"""
import numpy as np
import pytest

from oracle import np_oracle
from paper_2405_14430_b200 import ToyDiTCuda

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("L,hs,heads,p,N,M,W,S", [
    (4, 32, 4, 64, 1, 4, 1, 6),
    (4, 32, 4, 64, 4, 4, 1, 6),
    (4, 128, 4, 256, 2, 4, 1, 4),
    (2, 64, 2, 128, 2, 2, 0, 3),
])
def test_pipeline_vs_numpy(L, hs, heads, p, N, M, W, S):
    rng = np.random.default_rng(L * 1000 + hs + p)
    layers, cb = np_oracle.random_model(rng, L, hs, 4 * hs)
    x0 = rng.uniform(-1, 1, size=(p, hs))
    ref = np_oracle.run_pipefusion(layers, cb, heads, x0, S, N, M, W, 0.1)
    with ToyDiTCuda.from_weights(layers, cb, heads, p, workers=N) as m:
        out = m.run_pipefusion(x0, S, M, W, 0.1).final_x
    assert _rel(out, ref) < 1e-2
