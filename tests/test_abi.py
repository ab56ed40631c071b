"""The C-ABI library builds, loads and exports every symbol include/ppca.h declares (no GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "ppca.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[a-z_0-9]+\s*\*?\s+)+\**(ppca_[a-z_0-9]+)\s*\(", src, re.M)))


def test_header_declares_the_north_star_entry_points():
    names = _declared()
    for fn in ["ppca_generate", "ppca_prime_power", "ppca_prime_oja", "ppca_prime_eigengame", "ppca_refine",
               "ppca_eval"]:
        assert fn in names


def test_library_loads_and_exports_all_declared_symbols():
    import paper_2109_03709_b200 as P
    lib = P.load()
    out = subprocess.run(["nm", "-D", "--defined-only", P.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r" T (ppca_\w+)", out))
    declared = set(_declared())
    assert declared <= exported, f"missing: {sorted(declared - exported)}"
    assert declared == set(P.EXPORTS)
    assert P.ppca_abi_version() == 1
    assert P.ppca_status_string(6) == "subspace collapse"


def test_library_is_sm100a_and_uses_no_torch():
    import paper_2109_03709_b200 as P
    out = subprocess.run(["cuobjdump", "--list-elf", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    deps = subprocess.run(["ldd", P.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in deps


def test_ctx_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2109_03709_b200 as P
    with pytest.raises(P.PPCAError):
        P.ppca_ctx_create(0)
