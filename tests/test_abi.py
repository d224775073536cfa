"""C-ABI boundary checks that need no GPU: the product library exists, loads,
and exports every symbol the public headers declare; the Python mirror maps
status codes onto the reference's exception classes."""
import ctypes
import re
from pathlib import Path

import pytest

import paper_2405_14430_b200 as pf

ROOT = Path(__file__).resolve().parents[1]


def _declared(header: Path):
    text = header.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pf_[a-z_]+)\s*\(", text)))


def test_headers_declare_exported_list():
    declared = _declared(ROOT / "include" / "pipefusion_b200.h") + \
        _declared(ROOT / "include" / "pipefusion_b200_debug.h")
    assert sorted(declared) == sorted(pf.EXPORTED_SYMBOLS)


def test_library_loads_and_exports_every_symbol():
    assert pf.LIB_PATH.exists(), "run __graft_entry__.build() first"
    lib = pf.load_library()
    for name in pf.EXPORTED_SYMBOLS:
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.pf_version()


def test_library_is_sm100a_native():
    # the fatbin must carry sm_100a SASS with tcgen05 MMA and TMA instructions
    import shutil
    import subprocess
    cuobjdump = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([cuobjdump, "-sass", str(pf.LIB_PATH)], capture_output=True,
                         text=True, timeout=300).stdout
    assert "sm_100a" in out
    assert "UTCHMMA" in out      # tcgen05.mma
    assert "UTMALDG" in out      # TMA tensor loads
    assert "LDTM" in out         # tcgen05.ld (TMEM -> registers)


def test_status_mapping():
    with pytest.raises(pf.ValidationError):
        pf._raise(pf.PF_VALIDATION, "x is not divisible")
    with pytest.raises(pf.NumericError):
        pf._raise(pf.PF_NUMERIC, "non-finite activation")
    with pytest.raises(pf.CudaError):
        pf._raise(pf.PF_CUDA, "boom")
    pf._raise(pf.PF_OK, "")


def test_mlp_hidden_rounds_like_lround():
    assert pf.mlp_hidden_of(1152, 4.0) == 4608
    assert pf.mlp_hidden_of(5, 2.5) == 13   # 12.5 rounds away from zero
    assert pf.mlp_hidden_of(16, 2.0) == 32


def test_null_context_is_rejected_without_gpu():
    lib = pf.load_library()
    assert lib.pf_stage_count(None) == 0
    assert lib.pf_run_pipefusion(None, None, 0, 1, 1, 0, ctypes.c_double(0.1), None,
                                 None) == pf.PF_VALIDATION


def test_make_initial_latent_matches_reference_stream():
    # the product's host RNG (C ABI) is bitwise the reference's mt19937_64 stream
    from oracle import loader
    if not loader.RESTATEMENT_LIB.exists():
        loader.build(reference=False)
    import numpy as np
    a = pf.make_initial_latent(0, 64, 32)
    b = loader.Restatement().make_initial_latent(0, 64, 32)
    assert np.array_equal(a, b)
    with pytest.raises(pf.ValidationError):
        pf.make_initial_latent(0, 0, 32)
