"""CPU-side checks of the drop-in boundary: the extension builds for sm_100a,
loads without a GPU and exports every symbol include/swedg_b200.h declares.
No compute calls (there is no GPU here)."""
import ctypes
import os
import re

import pytest

from paper_2005_02516_b200 import build, capi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(REPO, "include", "swedg_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(swedg_[a-z0-9_]+)\s*\(", src)))


def test_extension_builds_for_sm100a():
    lib = build.build()
    assert os.path.exists(lib)
    out = os.popen(f"cuobjdump --list-elf {lib} 2>&1").read()
    assert "sm_100a" in out, out


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(build.build())
    names = header_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/swedg_b200.h but not exported"
    assert sorted(capi.EXPORTED) == names


def test_abi_version_and_create_error_without_gpu():
    lib = capi.lib()
    assert lib.swedg_abi_version() == capi.ABI_VERSION == 5
    # with no device, creation fails loudly (no CPU fallback)
    import torch

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(capi.SwedgError):
        capi.Handle(scheme=0, N=1, Np=3, nq=4, nf=6, npf=2, K=1, g=9.81, Qr=[0.0] * 100,
                    Qs=[0.0] * 100, wf=[1.0] * 6, gf=[0.0] * 40, sJ=[1.0] * 6, nx=[0.0] * 6,
                    ny=[0.0] * 6, nbr=[-1, -1, -1], perm=[0] * 6, Vq=[0.0] * 12, Vf=[0.0] * 18,
                    Pq=[0.0] * 12, Mh_inv=[0.0] * 9)
