"""CPU checks of the boundary: libadi.so builds, loads and exports every symbol
that include/adi.h declares; the product package has no CPU fallback and
never touches the oracle.  (No compute calls: there is no GPU here.)"""
import ast
import os
import re
import subprocess

import pytest

from conftest import ROOT

HEADER = os.path.join(ROOT, "include", "adi.h")
PKG = os.path.join(ROOT, "paper_2006_07583_b200")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(adi_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2006_07583_b200.build import build
    return build()


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("adi_create", "adi_set_source", "adi_set_boundary", "adi_step", "adi_get_fields"):
        assert n in names


def test_library_exports_every_declared_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (adi_[a-z_]+)\b", out))
    missing = [n for n in declared_functions() if n not in exported]
    assert not missing, missing


def test_library_loads_and_binding_names(libpath):
    import paper_2006_07583_b200 as adi
    L = adi.lib()
    for n in declared_functions():
        assert hasattr(L, n), n
        assert hasattr(adi, n), n   # the binding carries the same names
    assert "sm_100a" in adi.adi_version()


def test_library_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_device_means_error_not_fallback(libpath):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2006_07583_b200 as adi
    with pytest.raises(adi.AdiError) as e:
        adi.adi_create(17, 17, 1 / 16, 0.05, 1.0, adi.ADI_MFD)
    assert e.value.code == adi.ADI_ECUDA


def test_product_never_imports_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith(".py"):
                tree = ast.parse(open(os.path.join(dirpath, f)).read())
                for node in ast.walk(tree):
                    if isinstance(node, ast.Import):
                        assert not any(a.name.split(".")[0] == "oracle" for a in node.names)
                    if isinstance(node, ast.ImportFrom):
                        assert (node.module or "").split(".")[0] != "oracle"
            if f.endswith((".cu", ".cuh", ".h", ".cpp")):
                assert "oracle" not in open(os.path.join(dirpath, f)).read().lower()


def test_bad_arguments_rejected_before_device(libpath):
    import paper_2006_07583_b200 as adi
    for args in ((8, 17, 0.1, 0.05, 1.0, 0), (17, 17, -1.0, 0.05, 1.0, 0), (17, 17, 0.1, 0.05, 1.0, 7)):
        with pytest.raises(adi.AdiError) as e:
            adi.adi_create(*args)
        assert e.value.code == adi.ADI_EINVAL


def test_binding_constants_match_the_header():
    """Every enumerator of include/adi.h (methods, statuses, parameters, kernel kinds, dist
    modes) exists in the binding with the header's value -- no drift between the two."""
    import re
    import paper_2006_07583_b200 as adi
    text = open(os.path.join(ROOT, "include", "adi.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)   # (comments may mention names)
    found = 0
    for body in re.findall(r"enum\s*\w*\s*\{(.*?)\}", text, flags=re.S):
        for name, val in re.findall(r"(ADI_[A-Z0-9_]+)\s*=\s*(-?\d+)", body):
            assert hasattr(adi, name), f"binding lacks {name}"
            assert getattr(adi, name) == int(val), (name, getattr(adi, name), val)
            found += 1
    assert found >= 35, found
