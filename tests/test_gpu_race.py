"""Race detection by timing amplification (compute-sanitizer is closed on this pool).

tools/race_jitter.py runs every device path on fixed inputs with the product
library and with a test build (-DSK_RACE_JITTER) that sleeps a random
0-1 us in one thread of four at every synchronisation point (mbarrier waits
and arrivals of the TMA CH chunk, cp.async ring barriers, last-CTA
reductions, the cooperative CG grid barrier). All paths are deterministic by
construction, so the outputs must be bit-identical. The detector's own
sensitivity is pinned too: a build with the CH kernel's step-barrier wait
removed (-DSK_RACE_SELFTEST_DROP_STEP_WAIT) must be caught.
"""
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
AB = ROOT / "_ab"
TOOL = ROOT / "tools" / "race_jitter.py"


def _fresh(lib: Path) -> bool:
    if not lib.exists():
        return False
    srcs = list((ROOT / "paper_2205_03354_b200" / "csrc").glob("*")) + [ROOT / "include" / "sk_cuda.h"]
    return lib.stat().st_mtime >= max(f.stat().st_mtime for f in srcs)


def _build(name: str, *flags: str) -> Path:
    lib = AB / f"{name}.so"
    if not _fresh(lib):
        subprocess.run([sys.executable, str(ROOT / "tools" / "ab_build.py"), name, *flags], check=True,
                       capture_output=True, timeout=900)
    return lib


def _run(tmp: Path, name: str, lib: Path | None) -> Path:
    out = tmp / f"{name}.npz"
    cmd = [sys.executable, str(TOOL), "run", "--out", str(out)] + (["--lib", str(lib)] if lib else [])
    subprocess.run(cmd, check=True, capture_output=True, timeout=600)
    return out


def _same(a: Path, b: Path) -> tuple[bool, str]:
    r = subprocess.run([sys.executable, str(TOOL), "compare", str(a), str(b)], capture_output=True, text=True)
    return r.returncode == 0, r.stdout


def test_jittered_build_is_bit_identical(tmp_path):
    jit = _build("jitter", "-DSK_RACE_JITTER")
    ref = _run(tmp_path, "ref", None)
    for k in range(2):
        ok, log = _same(ref, _run(tmp_path, f"jit{k}", jit))
        assert ok, log


def test_detector_catches_a_dropped_wait(tmp_path):
    broken = _build("jitter_broken", "-DSK_RACE_JITTER", "-DSK_RACE_SELFTEST_DROP_STEP_WAIT")
    ref = _run(tmp_path, "ref", None)
    caught = False
    for k in range(3):  # the race is timing-dependent; amplified it shows within a run or two
        ok, log = _same(ref, _run(tmp_path, f"broken{k}", broken))
        if not ok:
            assert "ch3d_tma" in log
            caught = True
            break
    assert caught
