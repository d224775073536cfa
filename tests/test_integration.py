"""The drop-in boundary exercised from the reference's side.

integration/Makefile compiles the reference's own sources with
integration/backend_cuda.patch applied (Backend::Cuda, `ditsim execute
--backend cuda`) and links them against libpipefusion_b200.so. CPU tests: the
patched build still passes the reference's own executor and CLI suites
(test_execute.cpp, test_cli.cpp), so the patch and the CLI11 shim change
nothing for the CPU backends. GPU tests: Backend::Cuda against
Backend::Inline through the reference's API (integration/test_backend_cuda.cpp),
and the CLI's execute manifest (ditsim.cpp:280-325) under --backend cuda vs
--backend inline.
"""
import json
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
BUILD = ROOT / "integration" / "_build"

needs_build = pytest.mark.skipif(not (BUILD / "ditsim").exists(),
                                 reason="integration/_build not built (needs /root/reference)")


def _run(args, timeout=600):
    return subprocess.run(args, cwd=ROOT, capture_output=True, text=True, timeout=timeout)


@needs_build
def test_reference_executor_suite_passes_on_the_patched_build():
    r = _run([str(BUILD / "test_execute")])
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed" in r.stdout


@needs_build
def test_reference_cli_suite_passes_on_the_patched_cli():
    r = _run([str(BUILD / "test_cli")])
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed" in r.stdout


@needs_build
def test_cli_rejects_unknown_backends_with_exit_two():
    cfg = BUILD / "configs" / "reference_execute.cfg"
    r = _run([str(BUILD / "ditsim"), "--config", str(cfg), "execute", "--backend", "gpu"])
    assert r.returncode == 2 and "threads, inline or cuda" in r.stderr


C1_CFG = """[model]
layers = 4
hidden_size = 128
heads = 4
param_count = 786432
[workload]
seq_len = 256
diffusion_steps = {S}
warmup_steps = 1
step_size = 0.1
[cluster]
device_count = 2
device_flops = 1e12
link_bandwidth = 1e10
[plan]
strategy = pipefusion
patches = 4
"""


def _manifest(cfg, backend, *extra):
    r = _run([str(BUILD / "ditsim"), "--config", str(cfg), "execute", "--backend", backend,
              *extra])
    assert r.returncode == 0, r.stdout + r.stderr
    return json.loads(r.stdout)


@pytest.mark.gpu
@needs_build
def test_backend_cuda_through_the_reference_api():
    r = _run([str(BUILD / "test_backend_cuda")])
    assert r.returncode == 0, r.stdout + r.stderr
    assert "| 0 failed" in r.stdout


@pytest.mark.gpu
@needs_build
@pytest.mark.parametrize("which", ["cref", "c1_s4", "c1_s5"])
def test_cli_execute_manifest_cuda_vs_inline(which, tmp_path):
    if which == "cref":
        cfg = BUILD / "configs" / "reference_execute.cfg"
    else:
        cfg = tmp_path / f"{which}.cfg"
        cfg.write_text(C1_CFG.format(S=int(which[-1])))
    extra = ["--compare"]
    cpu = _manifest(cfg, "inline", *extra)
    gpu = _manifest(cfg, "cuda", *extra)
    # every manifest field the CLI writes, bar the measured ones, is identical
    keys = set(cpu) - {"divergence", "wall_time_s"}
    assert set(gpu) == set(cpu)
    assert {k: gpu[k] for k in keys} == {k: cpu[k] for k in keys}
    assert gpu["strategy"] == "compare" and gpu["divergence"]["serial"] == 0.0
    # divergences of the GPU strategies from the GPU serial oracle agree with
    # the fp64 ones (both are ~2-4e-2; the bf16 path moves them by < 5e-3)
    for k in ("pipefusion", "distrifusion"):
        assert abs(gpu["divergence"][k] - cpu["divergence"][k]) <= 5e-3, (k, gpu, cpu)
    assert gpu["wall_time_s"] > 0


@pytest.mark.gpu
@needs_build
def test_cli_execute_auto_warmup_and_trajectory_cuda(tmp_path):
    cfg = BUILD / "configs" / "reference_execute.cfg"
    cpu = _manifest(cfg, "inline", "--auto-warmup", "0.05",
                    "--dump-trajectory", str(tmp_path / "cpu.csv"))
    gpu = _manifest(cfg, "cuda", "--auto-warmup", "0.05",
                    "--dump-trajectory", str(tmp_path / "gpu.csv"))
    assert gpu["auto_warmup"] == cpu["auto_warmup"] == {"warmup": 16, "threshold_met": True}
    assert gpu["warmup"] == 16
    assert abs(gpu["divergence"] - cpu["divergence"]) <= 5e-3
    rows_c = (tmp_path / "cpu.csv").read_text().splitlines()
    rows_g = (tmp_path / "gpu.csv").read_text().splitlines()
    assert len(rows_g) == len(rows_c) == 21
    import numpy as np
    for a, b in zip(rows_c, rows_g):
        va, vb = (np.array([float(v) for v in r.split(",")]) for r in (a, b))
        assert va[0] == vb[0]  # step label
        assert np.linalg.norm(va[1:] - vb[1:]) <= 1e-2 * np.linalg.norm(va[1:])
    assert rows_c[0] == rows_g[0]  # the initial latent is dumped exactly
