"""The C-ABI boundary (CPU only, no compute calls): libouro_b200.so loads and
exports every function include/ouro.h declares; the oracle library exports
every function its header declares; the device header compiles into a user
program built from two translation units (examples/)."""
import ctypes as C
import os
import re
import subprocess

import pytest

import paper_2504_18211_b200 as ob
from oracle_lib import ORACLE_SO, oracle

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header, prefix):
    text = open(header).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(" + prefix + r"[a-z0-9_]+)\s*\(", text)))


def test_product_exports_every_declared_symbol():
    names = _declared(os.path.join(ROOT, "include", "ouro.h"), "ouro_")
    assert len(names) >= 30
    L = C.CDLL(ob.lib_path())
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_oracle_exports_every_declared_symbol():
    names = _declared(os.path.join(ROOT, "oracle", "ouro_oracle.hpp"), "orc_")
    oracle()
    L = C.CDLL(ORACLE_SO)
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_product_does_not_link_the_oracle():
    out = subprocess.run(["nm", "-D", "--defined-only", ob.lib_path()], capture_output=True, text=True).stdout
    assert "orc_" not in out
    ldd = subprocess.run(["ldd", ob.lib_path()], capture_output=True, text=True).stdout
    assert "oracle" not in ldd


def test_sm100a_code_present():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", ob.lib_path()],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_view_size_matches_header():
    # ouro_heap_view is passed by value to kernels; the C-ABI reports its size
    assert ob.lib().ouro_heap_view_size() >= 200


def test_user_program_builds():
    r = subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert os.path.exists(os.path.join(ROOT, "examples", "user_kernel"))


@pytest.mark.gpu
def test_user_program_runs(cuda):
    exe = os.path.join(ROOT, "examples", "user_kernel")
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "examples")], check=True)  # rebuild if headers changed
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.strip().endswith("ok")
