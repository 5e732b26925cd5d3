"""build.py's rebuild rule (CPU, no nvcc): an object is rebuilt when its
sources are newer or when its nvcc command line changed, so an experiment
build (QGS_NVCC_EXTRA) is never taken for the product."""

import os
import subprocess

from paper_2411_16392_b200 import build as b


def _fake_tree(tmp_path, monkeypatch):
    csrc = tmp_path / "csrc"
    inc = tmp_path / "include"
    csrc.mkdir()
    inc.mkdir()
    (inc / "qgs_b200.h").write_text("// header\n")
    (csrc / "a.cuh").write_text("// shared\n")
    units = {"one.cu": ["-fmad=false"], "two.cu": []}
    for u in units:
        (csrc / u).write_text(f"// {u}\n")
    monkeypatch.setattr(b, "CSRC", str(csrc))
    monkeypatch.setattr(b, "INCLUDE", str(inc))
    monkeypatch.setattr(b, "UNITS", units)
    monkeypatch.setattr(b, "nvcc", lambda: "nvcc")
    calls = []

    def fake_call(cmd):
        calls.append(cmd)
        out = cmd[cmd.index("-o") + 1]
        with open(out, "w") as f:
            f.write(" ".join(cmd))
        return 0

    monkeypatch.setattr(subprocess, "check_call", fake_call)
    return csrc, calls


def _compiles(calls):
    return [c for c in calls if "-c" in c]


def test_rebuild_on_flags_and_sources(tmp_path, monkeypatch):
    csrc, calls = _fake_tree(tmp_path, monkeypatch)
    obj, lib = str(tmp_path / "obj"), str(tmp_path / "lib.so")
    monkeypatch.delenv("QGS_NVCC_EXTRA", raising=False)

    b._build(obj, lib, [], False, False)
    assert len(_compiles(calls)) == 2 and os.path.exists(lib)

    calls.clear()
    b._build(obj, lib, [], False, False)          # nothing changed
    assert calls == []

    calls.clear()
    monkeypatch.setenv("QGS_NVCC_EXTRA", "-DQGS_EXPERIMENT=1")
    b._build(obj, lib, [], False, False)          # experiment flags: everything
    assert len(_compiles(calls)) == 2
    assert all("-DQGS_EXPERIMENT=1" in c for c in _compiles(calls))

    calls.clear()
    monkeypatch.delenv("QGS_NVCC_EXTRA")
    b._build(obj, lib, [], False, False)          # back to the product flags
    assert len(_compiles(calls)) == 2
    assert not any("-DQGS_EXPERIMENT=1" in c for c in calls)

    calls.clear()
    src = csrc / "two.cu"
    later = os.path.getmtime(src) + 20
    for o in os.listdir(obj):                     # objects newer than every source ...
        os.utime(os.path.join(obj, o), (later - 10, later - 10))
    os.utime(src, (later, later))                 # ... except two.cu
    b._build(obj, lib, [], False, False)          # one newer source: that unit + link
    comp = _compiles(calls)
    assert len(comp) == 1 and comp[0][-3].endswith("two.cu")
    assert any("-shared" in c for c in calls)
