"""The C-ABI library loads without a GPU and exports every symbol the headers declare; calls
that need a device fail loudly (no CPU fallback)."""
import os
import re
import subprocess

import pytest

import paper_2504_21440_b200 as q

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    txt = open(os.path.join(ROOT, "include", header)).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return set(re.findall(r"\b(qsg_[a-z_0-9]+)\s*\(", txt))


def exported():
    out = subprocess.run(["nm", "-D", "--defined-only", q.LIB_PATH], capture_output=True, text=True).stdout
    return {l.split()[-1] for l in out.splitlines() if " T " in l}


@pytest.mark.parametrize("header", ["qsg.h", "qsg_model.h"])
def test_every_declared_symbol_is_exported(header):
    names = declared(header)
    assert len(names) >= 8
    missing = names - exported()
    assert not missing, missing


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", q.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    with pytest.raises(q.QsgError) as e:
        q.Context(0)
    assert e.value.code == 100


def test_host_api_reports_library_errors():
    with pytest.raises(q.QsgError) as e:
        q.Model("kerr", 0, 1.0, 0.1, 0.1, 0.1)  # InvalidDimension (factories.cpp:18-20)
    assert e.value.code == 4
