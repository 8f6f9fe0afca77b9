"""CPU-side checks of the C-ABI boundary: the libraries build for sm_100a,
load, and export every symbol include/snp.h declares; the binding fails
loudly (no CPU fallback) when no GPU is present.  No compute calls."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def built():
    from paper_1104_1824_b200 import build
    build.build()
    return build


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "snp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(snp_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("snp_load", "snp_step", "snp_explore", "snp_begin", "snp_advance", "snp_tree_configs"):
        assert s in syms


def test_library_exports_every_declared_symbol(built):
    lib = ctypes.CDLL(built.LIB_SNP)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    out = subprocess.check_output(["nm", "-D", "--defined-only", built.LIB_SNP]).decode()
    for s in declared_symbols():
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_binding_names_match_header(built):
    from paper_1104_1824_b200 import snp
    assert sorted(snp.EXPORTED) == declared_symbols()


def test_sm100a_code_present(built):
    out = subprocess.check_output(["/usr/local/cuda/bin/cuobjdump", "--list-elf", built.LIB_SNP]).decode()
    assert "sm_100a" in out


def test_abi_version(built):
    lib = ctypes.CDLL(built.LIB_SNP)
    assert lib.snp_abi_version() == 2  # round 2: keep_all_edges, overflow_fixes fields


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback(built):
    from paper_1104_1824_b200 import snp
    from paper_1104_1824_b200 import workloads as W
    with pytest.raises(snp.SnpError) as e:
        snp.System(W.pi_system("simulator"))
    assert e.value.status == snp.SNP_E_CUDA


def test_engine_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1104_1824_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "oracle.h" not in txt, f
