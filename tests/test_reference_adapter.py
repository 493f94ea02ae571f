"""The reference-side drop-in (include/marl_b200_vector_env.hpp) compiles
against the UNMODIFIED reference headers, links both the reference library
and libmarl_b200.so, and translates engine statuses into the reference's
exception taxonomy.  Built here only (needs /root/reference); on a machine
without a GPU the constructor must raise instead of falling back to the CPU.
With a GPU (`-m gpu`), the adapter's reset/step must equal the reference
VectorEnv's bit for bit on SMAX."""
from __future__ import annotations

import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/core/include"
JSON_DIR = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann"
LIB = os.path.join(ROOT, "paper_2311_10090_b200", "_lib", "libmarl_b200.so")
REF_LIB = os.path.join(ROOT, "oracle", "_ref", "libmarl_ref.so")

SRC = os.path.join(ROOT, "oracle", "adapter_parity.cpp")
PREBUILT = os.path.join(ROOT, "oracle", "_ref", "adapter_parity")


def _build(tmp_path):
    if not os.path.isdir(REF_INC) or not os.path.exists(REF_LIB):
        pytest.skip("reference headers / oracle/_ref not available on this machine")
    if not os.path.exists(LIB):
        pytest.skip("libmarl_b200.so not built")
    exe = tmp_path / "adapter"
    cmd = ["g++", "-std=c++20", "-O1", "-I", REF_INC, "-I", JSON_DIR, "-I", os.path.join(ROOT, "include"),
           SRC, "-o", str(exe), REF_LIB, LIB, f"-Wl,-rpath,{os.path.dirname(LIB)}",
           f"-Wl,-rpath,{os.path.dirname(REF_LIB)}", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return exe


def test_adapter_compiles_and_refuses_without_gpu(tmp_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("covered by the -m gpu parity variant")
    exe = _build(tmp_path)
    r = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1 and "runtime_error" in r.stdout, r.stdout + r.stderr


@pytest.mark.gpu
def test_adapter_matches_reference_vectorenv():
    """Prebuilt by __graft_entry__.build() (oracle/Makefile `adapter`)."""
    if not os.path.exists(PREBUILT):
        pytest.skip("oracle/_ref/adapter_parity not built (needs the reference headers at build time)")
    r = subprocess.run([PREBUILT], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ADAPTER PARITY OK" in r.stdout, r.stdout + r.stderr
