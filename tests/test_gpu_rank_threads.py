"""The rank >= 0 distributed code path (not the rank = -1 emulation) on one GPU.

Ranks are threads of one process; the NCCL entry points come from the
in-process shim tests/nccl_shim/msk_nccl_shim.cpp through libmsk's
MSK_NCCL_LIBRARY hook.  The shim turns a collective issued by fewer ranks, a
mismatched count / datatype or an unmatched receive into an error, i.e. what
would deadlock or corrupt a real NCCL job.  Every rank must reproduce the
single-GPU alpha, iteration counts and s_L bit for bit.

The CPU part compiles the shim and checks that it exports every NCCL entry
point libmsk resolves (paper_2503_04914_b200/csrc/nccl_dl.cuh).
"""
import os
import re
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHIM_SRC = os.path.join(ROOT, "tests", "nccl_shim", "msk_nccl_shim.cpp")
SHIM_DIR = os.path.join(ROOT, "tests", "nccl_shim", "_build")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def build_shim() -> str:
    os.makedirs(SHIM_DIR, exist_ok=True)
    out = os.path.join(SHIM_DIR, "libmsk_nccl_shim.so")
    cmd = ["g++", "-O2", "-std=c++17", "-shared", "-fPIC", "-I", os.path.join(CUDA, "include"), SHIM_SRC,
           "-o", out, os.path.join(CUDA, "lib64", "libcudart_static.a"), "-ldl", "-lpthread", "-lrt"]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return out


def test_shim_builds_and_exports_every_resolved_symbol():
    lib = build_shim()
    syms = subprocess.run(["nm", "-D", "--defined-only", lib], check=True, capture_output=True,
                          text=True).stdout
    with open(os.path.join(ROOT, "paper_2503_04914_b200", "csrc", "nccl_dl.cuh")) as fh:
        wanted = set(re.findall(r'sym\("(nccl\w+)"\)', fh.read()))
    assert len(wanted) == 10
    have = set(re.findall(r" T (nccl\w+)", syms))
    assert wanted <= have, wanted - have


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3, 4])
def test_rank_threads_equal_single_gpu_bitwise(world):
    lib = build_shim()
    env = dict(os.environ, MSK_NCCL_LIBRARY=lib, MSK_SHIM_TIMEOUT_S="60")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "nccl_shim", "threads_dist.py"), str(world)],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]


@pytest.mark.gpu
def test_rank_threads_full_size_bench_configuration():
    """C3 as bench.py --gpus 2 runs it (the levels the latency model partitions:
    the 1.25M and 10M levels), 10^6 evaluation points: both ranks bit-identical
    to the single-GPU solve."""
    lib = build_shim()
    env = dict(os.environ, MSK_NCCL_LIBRARY=lib, MSK_SHIM_TIMEOUT_S="120")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "nccl_shim", "threads_dist.py"), "2", "--full"],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0 and "ALL OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
