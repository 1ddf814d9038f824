"""The C ABI library loads, exports every entry point include/smap.h declares,
and validates arguments on the host without touching a GPU.  CPU only."""
import ctypes
import re
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def sm():
    import paper_1610_07394_b200 as s
    return s


def test_header_symbols_exported(sm):
    lib = ctypes.CDLL(sm.LIB_PATH)
    names = sm.exported_symbols()
    assert {"smap_plan", "smap_run", "smap_run_host", "smap_destroy", "smap_stats_fetch", "smap_out_bytes",
            "smap_volume", "smap_last_error", "smap_plan_query", "smap_abi_version"} <= set(names)
    for name in names:
        assert hasattr(lib, name), name


def test_header_is_plain_c():
    src = open(os.path.join(ROOT, "include", "smap.h")).read()
    assert 'extern "C"' in src
    assert not re.search(r"\btorch\b|\bat::|\bc10::", src)


def test_abi_version(sm):
    assert sm.smap_abi_version() == 1


def test_volume(sm):
    assert sm.smap_volume(2, 4) == 6
    assert sm.smap_volume(2, 4, "inclusive") == 10
    assert sm.smap_volume(3, 1024) == 178433024
    assert sm.smap_volume(2, 1 << 17) == 8589869056
    assert sm.smap_volume(3, 2048) == 1429559296


@pytest.mark.parametrize("kw", [dict(m=4, n=64, rho=8), dict(m=2, n=100, rho=3), dict(m=2, n=64, rho=128),
                                dict(m=2, n=1, rho=1), dict(m=3, n=2, rho=1), dict(m=2, n=64, rho=8, shard_count=3),
                                dict(m=2, n=1024, rho=16, granularity="tile"), dict(m=3, n=32, rho=8),
                                dict(m=2, n=64, rho=8, map="bb", shard_count=2)])
def test_invalid_plans_rejected_before_device_work(sm, kw):
    with pytest.raises(sm.SmapError) as e:
        sm.smap_plan(**kw)
    assert e.value.status == 1
    assert sm.smap_last_error()


def test_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1610_07394_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                for bad in ("import oracle", "from oracle", "liboracle", "oracle.c", "or_lambda"):
                    assert bad not in src, (f, bad)
