"""CPU checks of the boundary: libsrl.so builds for sm_100a, loads, and exports every entry
point include/srl.h declares; host-side validation rejects bad arguments without a GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "srl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(srl_[a-z_0-9]+)\s*\(", src)))


@pytest.fixture(scope="module")
def L():
    from paper_2306_16688_b200 import build
    build.build()
    import paper_2306_16688_b200 as P
    return P.lib()


def test_exports_every_declared_symbol(L):
    names = _declared()
    assert "srl_gae" in names and "srl_ppo_step" in names and "srl_allreduce_grads" in names
    for n in names:
        assert hasattr(L, n), n
    import paper_2306_16688_b200 as P
    assert sorted(P.EXPORTS) == names


def test_abi_version(L):
    assert L.srl_abi_version() == 3


def test_sass_is_sm100a_tcgen05():
    """The built library carries sm_100a SASS with tcgen05 MMA, TMEM loads and TMA."""
    import shutil
    import subprocess
    cu = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    so = os.path.join(ROOT, "paper_2306_16688_b200", "libsrl.so")
    out = subprocess.run([cu, "-sass", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out or "SM100" in out.upper()
    assert "UTCHMMA" in out or "UTCMMA" in out
    assert "LDTM" in out and "UTMALDG" in out


def test_validation_without_gpu(L):
    # null pointers / bad shapes are rejected on the host before any launch
    assert L.srl_gae(0, 4, 4, None, None, None, None, None, 0.99, 0.95, None, None, None, None) == 1
    assert L.srl_gae(8, 4, 4, None, None, None, None, None, 0.99, 0.95, None, None, None, None) == 1
    assert b"srl_gae" in L.srl_last_error()
    assert L.srl_ppo_step(None, 1, 1, None, None, None, None, None, None, None, None, 1, None, None) == 1
    assert L.srl_allreduce_grads(None, None, 0, 0, None) == 1


def test_create_rejects_bad_config(L):
    import paper_2306_16688_b200.srl as S
    hid = (C.c_int * 1)(100)      # not a multiple of 64
    heads = (C.c_int * 1)(2)
    cfg = S.PPOConfigC(4, 8, 1, hid, 1, heads, 0.2, 0.5, 0.01, 3e-4, 0.9, 0.999, 1e-8, 1e-8,
                       0.99, 0.95, 0, 32, 0, 0.0, 0.0, 1, 1, 0)
    h = C.c_void_p()
    assert L.srl_ppo_create(C.byref(cfg), 0, 1, None, 0, C.byref(h)) == 1
    assert b"hidden" in L.srl_last_error()
