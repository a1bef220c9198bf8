"""CPU-side checks of the C-ABI boundary (no compute calls without a GPU).

* libmsk.so builds for sm_100a and loads;
* it exports every entry point include/msk.h declares;
* the Python binding mirrors them by name;
* without a usable CUDA device the library fails loudly (no CPU fallback).
"""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    with open(os.path.join(ROOT, "include", "msk.h")) as fh:
        text = fh.read()
    return sorted(set(re.findall(r"MSK_API\s+[\w\s\*]*?\b(msk_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2503_04914_b200 import build
    build.build()
    import paper_2503_04914_b200 as m
    return m.load()


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("msk_ctx_create", "msk_hierarchy_create", "msk_assemble", "msk_solve",
                 "msk_evaluate", "msk_hierarchy_destroy", "msk_ctx_destroy", "msk_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    so = os.path.join(ROOT, "paper_2503_04914_b200", "libmsk.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(msk_\w+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    for n in _declared():
        assert hasattr(lib, n)


def test_binding_mirrors_names(lib):
    import paper_2503_04914_b200 as m
    for n in _declared():
        assert callable(getattr(m, n)), n


def test_sm100a_code_present():
    so = os.path.join(ROOT, "paper_2503_04914_b200", "libmsk.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_no_oracle_in_product_path():
    """The product package never imports or links the oracle."""
    pkg = os.path.join(ROOT, "paper_2503_04914_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                with open(os.path.join(dirpath, f)) as fh:
                    src = fh.read()
                assert "oracle" not in re.sub(r"//.*|#.*|\"\"\"[\s\S]*?\"\"\"", "", src).lower() or \
                    "import oracle" not in src, f


def test_fails_loudly_without_gpu(lib):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_2503_04914_b200 as m
    with pytest.raises(m.MskError) as ei:
        m.Context(0)
    assert ei.value.status in (1, 3)
    assert m.msk_version().startswith("libmsk")


def _build_c_example(tmp_path):
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    libdir = os.path.join(root, "paper_2503_04914_b200")
    exe = str(tmp_path / "msk_example")
    subprocess.check_call(["gcc", "-std=c99", "-O2", "-Wall", "-Wextra", "-Werror",
                           os.path.join(root, "examples", "msk_example.c"), "-I", os.path.join(root, "include"),
                           "-L", libdir, "-lmsk", f"-Wl,-rpath,{libdir}", "-lm", "-o", exe])
    return exe


def test_c_example_builds_and_fails_loudly_without_gpu(tmp_path):
    """include/msk.h is plain C99 and libmsk links from C; without a usable
    device the first call reports MSK_ERR_CUDA (no CPU path)."""
    import subprocess
    import torch
    exe = _build_c_example(tmp_path)
    if torch.cuda.is_available():
        pytest.skip("a GPU is present (tests/test_gpu_parity.py runs the example)")
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 2 and "msk_ctx_create" in r.stderr
