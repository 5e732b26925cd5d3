"""Memory safety of every CUDA path under the bounds-checking build.

compute-sanitizer is closed on the GPU pool, so the library is also built
with QGS_DEBUG_CHECKS=1 (libqgs_b200_debug.so: device checks of every
shared-memory queue, ring, fragment-log page, sort rank and bucket slot;
a failed check traps the kernel) and tools/sanitize_view.py drives every
path through it -- prepare, forward (exact / fp32 decisions, resort off,
Euclidean density, a page pool that runs dry), backward (atomics,
deterministic, log and replay), chain, the PreparedView exports -- on C1 and
on a reduced degenerate C5 view.  The results must also still match the
product build's.
"""

import os
import subprocess
import sys

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def _run(variant, *args):
    env = dict(os.environ)
    if variant:
        env["QGS_LIB_VARIANT"] = variant
    out = subprocess.run([sys.executable, os.path.join(REPO, "tools", "sanitize_view.py"), *args],
                         capture_output=True, text=True, timeout=900, cwd=REPO, env=env)
    assert out.returncode == 0, (out.stdout[-2000:], out.stderr[-3000:])
    assert "QGS_CHECK failed" not in out.stdout + out.stderr
    return out.stdout


@pytest.mark.parametrize("args", [("--config", "c1"), ("--config", "c5", "--n", "20000", "--res", "192")])
def test_every_path_under_bounds_checks(cuda_device, args):
    dbg = _run("debug", *args)
    assert "lib libqgs_b200_debug.so" in dbg
    ref = _run(None, *args)
    # the same pair count and (deterministic) forward maps, bit for bit; the
    # deterministic backward to rounding (the check branches change how the
    # compiler contracts a few products)
    assert dbg.splitlines()[-1] == ref.splitlines()[-1]
    d, r = (float(ln.split()[1]) for ln in (dbg.splitlines()[-2], ref.splitlines()[-2]))
    assert abs(d - r) <= 1e-6 * abs(r)
