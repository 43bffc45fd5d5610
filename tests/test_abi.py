"""CPU: the C-ABI library loads and exports every symbol include/distgrid_b200.h declares
(no compute calls — this container has no GPU)."""
import ctypes as C
import os

import pytest

from paper_2405_04416_b200 import abi, dg


def test_library_built_for_sm100a():
    assert os.path.exists(dg.LIB_PATH), "run __graft_entry__.build()"
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", dg.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_exports_every_header_symbol():
    L = dg.lib()
    names = dg.header_functions()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_struct_sizes_match_header():
    # sizes the C side expects (checked against offsets of trailing fields)
    assert C.sizeof(abi.RunConfig) == 320
    assert C.sizeof(abi.RayBatch) == 56
    assert C.sizeof(abi.StepStats) == 112
    assert C.sizeof(abi.Merged) == 40


def test_default_config_matches_reference_defaults():
    c = abi.RunConfig()
    dg.lib().dg_default_config(C.byref(c))
    d = abi.default_config()
    for name, _ in abi.RunConfig._fields_:
        a, b = getattr(c, name), getattr(d, name)
        if hasattr(a, "__len__"):
            assert list(a) == list(b), name
        else:
            assert a == b, name


def test_lr_schedule_matches_oracle():
    from oracle.bindings import oracle_lib
    c = abi.default_config()
    c.total_steps = 1000
    for s in (0, 1, 17, 500, 999, 1000):
        assert dg.lr_at(c, s) == oracle_lib().or_lr_at(C.byref(c), s)


def test_error_mapping_on_bad_config():
    # configuration validation happens before any device work and maps to DG_EINVAL
    c = abi.default_config()
    c.grid_features = 4
    with pytest.raises(dg.DGError) as e:
        dg.Context(c, device=0)
    assert e.value.status in ("DG_EINVAL", "DG_ECUDA")


@pytest.mark.parametrize("src", ["tests/cpp/facade_demo.cpp", "tests/cpp/facade_stages.cpp"])
def test_facade_headers_compile(src):
    """The C++ facade (include/distgrid/*.hpp) compiles as a reference user's code would."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run(["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-I", os.path.join(root, "include"),
                        os.path.join(root, src)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-3000:]
