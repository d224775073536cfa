"""bench.py's reference arm on the CPU (what the driver runs as
`bench.py --impl reference`): the reference's own implementation timed on
the host, printed as one JSON line with the contract's keys and the same
`config` as the GPU arm."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _line(*args):
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", *args],
                       capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])


@pytest.mark.parametrize("cfg", ["cref", "c1"])
def test_reference_arm_small_configs_run_the_full_image(cfg):
    d = _line("--config", cfg, "--steps", "1", "--warmup", "1", "--cpu-budget", "30")
    assert d["impl"] == "reference" and d["higher_is_better"] is False
    assert d["unit"] == "s/image" and d["value"] > 0
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "reference"
    assert "one full image" in d["cpu_baseline"]["sample"]
    import bench  # noqa: F401  (same config keys as the GPU arm)
    assert d["config"] == bench.config_of(bench.CONFIGS[cfg], 1, 1)


def test_reference_arm_c2_is_a_bounded_extrapolated_sample():
    d = _line("--steps", "1", "--warmup", "1", "--cpu-budget", "2")
    base = d["cpu_baseline"]
    assert base["kind"] == "reference" and "extrapolated" in base["sample"]
    assert base["single_thread_value"] >= base["value"] > 1000  # hours of CPU per C2 image
    assert d["config"]["seq_len"] == 4096 and d["config"]["layers"] == 28
