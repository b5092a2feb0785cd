"""CPU tests of the C-ABI library: it loads, exports every symbol declared in
include/gpair.h, and its host-only functions behave (no GPU compute here)."""
import ctypes
import math
import os
import re

import pytest

from oracle import ir
from paper_2602_03893_b200 import gpair
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "gpair.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gpair_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2602_03893_b200 import build

    build.build()
    return gpair.lib()


def test_every_declared_symbol_is_exported(lib):
    names = _declared_functions()
    assert len(names) >= 14, names
    raw = ctypes.CDLL(gpair.LIB_PATH)
    missing = [n for n in names if not hasattr(raw, n)]
    assert not missing, missing


def test_struct_layouts_match_header(lib, tmp_path):
    """ctypes mirrors have the C sizes and field offsets (compiled with gcc)."""
    import subprocess

    structs = {"gpair_desc": gpair.Desc, "gpair_step": gpair.Step, "gpair_profile": gpair.Profile,
               "gpair_info": gpair.Info}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "gpair.h"', "int main(void){"]
    for cname, cls in structs.items():
        lines.append(f'printf("{cname} %zu\\n", sizeof({cname}));')
        for f, _ in cls._fields_:
            lines.append(f'printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    lines.append("return 0;}")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    out = dict(l.split() for l in subprocess.check_output([str(exe)], text=True).splitlines())
    for cname, cls in structs.items():
        assert int(out[cname]) == ctypes.sizeof(cls), cname
        for f, _ in cls._fields_:
            assert int(out[f"{cname}.{f}"]) == getattr(cls, f).offset, (cname, f)


def test_cawr_host_function_matches_eq24(lib):
    for t in range(0, 230, 3):
        for Tm in (1, 2, 3):
            for printed in (True, False):
                a = gpair.cawr_lr(t, 1e-4, 0.1, 50, Tm, printed)
                b = ir.cawr(t, 1e-4, 0.1, 50, Tm, printed)
                assert a == pytest.approx(b, rel=1e-13, abs=1e-16), (t, Tm, printed)
    assert math.isnan(gpair.cawr_lr(-1, 0, 1, 50, 1))
    assert math.isnan(gpair.cawr_lr(3, 0, 1, 0, 1))


def test_strerror_and_version(lib):
    assert lib.gpair_strerror(0) == b"ok"
    assert lib.gpair_strerror(2) == b"geometry conflict"
    assert b"sm_100a" in lib.gpair_version()


def test_create_validates_before_touching_the_device(lib):
    d = gpair.Desc(sound_speed=1500.0, sampling_rate=40e6, n_samples=64, t0=0.0, n_kernels=8, centers=1,
                   sigma=0.0, sigmas=None, window_k=3.0, n_sensors=4, sensors=1, rank=0, world=1, nccl_comm=None,
                   flags=0)
    h = ctypes.c_void_p()
    assert lib.gpair_create(ctypes.byref(h), ctypes.byref(d), None) == gpair.ERR_INVALID_ARGUMENT
    assert b"sigma" in lib.gpair_last_error(None)
    assert not h.value
    d.sigma = 1e-4
    d.n_samples = 0
    assert lib.gpair_create(ctypes.byref(h), ctypes.byref(d), None) == gpair.ERR_INVALID_ARGUMENT
    d.n_samples = 64
    d.sigmas = 1  # per-kernel sigma (row f4) needs the exact operator, not ASSA
    d.flags = gpair.TOF_ASSA
    assert lib.gpair_create(ctypes.byref(h), ctypes.byref(d), None) == gpair.ERR_INVALID_ARGUMENT
    d.sigmas = None
    d.flags = gpair.TOF_ASSA | gpair.NEAR_FIELD
    assert lib.gpair_create(ctypes.byref(h), ctypes.byref(d), None) == gpair.ERR_INVALID_ARGUMENT
    d.flags = 0
    d.world = 2
    assert lib.gpair_create(ctypes.byref(h), ctypes.byref(d), None) == gpair.ERR_INVALID_ARGUMENT
    d.world = 1
    d.n_sensors = 1 << 20
    d.n_samples = 1 << 12
    assert lib.gpair_create(ctypes.byref(h), ctypes.byref(d), None) == gpair.ERR_RESOURCE
    assert lib.gpair_create(None, ctypes.byref(d), None) == gpair.ERR_INVALID_ARGUMENT
    assert lib.gpair_forward(None, None, None, None) == gpair.ERR_INVALID_ARGUMENT
    assert lib.gpair_destroy(None) == 0


def test_product_package_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2602_03893_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(import oracle|from oracle)", txt, flags=re.M), f
                assert not re.search(r'#\s*include\s*[<"][^>"]*oracle', txt), f
                assert "liboracle" not in txt, f
