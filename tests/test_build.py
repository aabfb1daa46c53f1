"""CPU-side checks of the CUDA boundary: the library builds for sm_100a, exports every
symbol include/zkdl.h declares, its hard-coded constants are right, and it refuses to
run without a device (no CPU fallback)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = 0x73EDA753299D7D483339D80809A1D80553BDA402FFFE5BFEFFFFFFFF00000001


@pytest.fixture(scope="module")
def so():
    from paper_2307_16273_b200 import build
    return build.build(verbose=False)


def test_exports_every_declared_symbol(so):
    from paper_2307_16273_b200 import _lib
    names = _lib.declared_symbols()
    assert len(names) >= 20
    L = ctypes.CDLL(so)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (zk_\w+)", out))
    assert set(names) <= exported


def test_sass_is_sm100a(so):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _limbs(x):
    return [(x >> (32 * i)) & 0xFFFFFFFF for i in range(8)]


def test_device_constants():
    txt = open(os.path.join(ROOT, "paper_2307_16273_b200", "csrc", "fr.cuh")).read()
    txt += open(os.path.join(ROOT, "paper_2307_16273_b200", "csrc", "transcript.cuh")).read()

    def grab(name):
        m = re.search(r"#define " + name + r"\s+fr_const\(([^)]*)\)", txt)
        return [int(v.strip().rstrip("u"), 16) for v in m.group(1).split(",")]
    R = 1 << 256
    assert grab("ZK_ONE") == _limbs(R % P)
    assert grab("ZK_R2") == _limbs(R * R % P)
    assert grab("ZK_R3") == _limbs(R ** 3 % P)
    assert grab("ZK_TWO31_MONT") == _limbs((1 << 31) * R % P)
    assert grab("ZK_INV2") == _limbs(pow(2, -1, P) * R % P)
    assert grab("ZK_INV6") == _limbs(pow(6, -1, P) * R % P)
    pl = [int(re.search(rf"#define ZK_P{i} (0x[0-9a-f]+)u", txt).group(1), 16) for i in range(8)]
    assert pl == _limbs(P)
    assert (-pow(P, -1, 1 << 32)) % (1 << 32) == 0xFFFFFFFF


def test_no_cpu_fallback():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2307_16273_b200 import api
    with pytest.raises(Exception):
        api.Context(0)
