"""The C ABI library loads, exports every entry point include/smap.h declares,
and validates arguments on the host without touching a GPU.  CPU only."""
import ctypes
import re
import math
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
    assert sm.smap_abi_version() == 2


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


def test_extreme_sizes_host_plans(sm):
    """Largest and smallest domains: closed forms exact in 64 bits (Python ints
    as the reference), u64 elements above 2^32, one-launch grid limits."""
    import math
    N = sm.DEVICE_NONE
    n = 1 << 30
    for diag, V in (("strict", math.comb(n, 2)), ("inclusive", n * (n + 1) // 2)):
        assert sm.smap_volume(2, n, diag) == V
        plan = sm.smap_plan(2, n, 512, diag=diag, granularity="tile", device=N, layout="tiles")
        q = sm.smap_plan_query(plan)
        assert q["useful_elems"] == V and q["launched_threads"] == q["grid_blocks"] * 512 ** 2
        assert sm.smap_out_bytes(plan, "index_write") == 8 * V          # u64 ranks beyond 2^32
        assert sm.smap_out_bytes(plan, "edm") == 4 * V
    assert sm.smap_volume(3, 1 << 21) == math.comb(1 << 21, 3)
    # a THREAD grid beyond one launch (2^31 - 1 blocks) is refused on the host
    with pytest.raises(sm.SmapError) as e:
        sm.smap_plan(2, 1 << 17, 2, map="bb", device=N)                  # 2^32 blocks
    assert e.value.status == 1
    sm.smap_plan(2, 1 << 16, 2, map="lambda", device=N)                  # 2^29 blocks: fine
    # smallest domains: one pair, one triple, one inclusive triple
    assert sm.smap_volume(2, 2) == 1 and sm.smap_volume(3, 3) == 1 and sm.smap_volume(3, 1, "inclusive") == 1
    for m, n_, d in ((2, 2, "strict"), (3, 3, "strict"), (3, 1, "inclusive"), (2, 1, "inclusive")):
        q = sm.smap_plan_query(sm.smap_plan(m, n_, 1, map="bb", diag=d, device=N))
        assert q["useful_elems"] == sm.smap_volume(m, n_, d)


def _build_c_example(tmp_path):
    import subprocess
    exe = str(tmp_path / "edm_c_api")
    pkg = os.path.join(ROOT, "paper_1610_07394_b200")
    cmd = ["gcc", "-O2", "-ffp-contract=off", "-I", os.path.join(ROOT, "include"), "-I", "/usr/local/cuda/include",
           os.path.join(ROOT, "examples", "edm_c_api.c"), "-L", pkg, "-lsmap", "-L", "/usr/local/cuda/lib64",
           "-lcudart", "-lm", f"-Wl,-rpath,{pkg}", "-o", exe]
    subprocess.run(cmd, check=True, capture_output=True)
    return exe


def test_c_example_compiles_against_the_header(tmp_path):
    """The boundary is a plain C ABI: examples/edm_c_api.c (C, no Python)
    compiles and links against include/smap.h and libsmap.so."""
    assert os.path.exists(_build_c_example(tmp_path))


def test_result_combine_and_locate_reject_bad_arguments(sm):
    """Argument checks of smap_result_combine / smap_locate / smap_run happen
    before any device work (so they run here, without a GPU)."""
    import ctypes as C
    lib = sm._lib
    buf = (C.c_int64 * 16)()
    assert lib.smap_result_combine(None, 1, C.cast(buf, C.c_void_p), None) == sm.E_INVALID
    assert lib.smap_result_combine(C.cast(buf, C.c_void_p), 0, C.cast(buf, C.c_void_p), None) == sm.E_INVALID
    misaligned = C.c_void_p(C.addressof(buf) + 4)
    assert lib.smap_result_combine(misaligned, 1, C.cast(buf, C.c_void_p), None) == sm.E_INVALID
    assert "aligned" in sm.smap_last_error()
    plan = sm.smap_plan(2, 1000, 32, map="below", granularity="tile", layout="tiles", device=sm.DEVICE_NONE)
    with pytest.raises(sm.SmapError):
        sm.smap_locate(plan, 5, 7)                       # j > i: outside the strict domain
    with pytest.raises(sm.SmapError):
        sm.smap_run(plan, "edm")                         # host-only plan cannot run
    # m=3 counts that would wrap 64 bits are refused at plan time (n = 2^22, 2^23)
    for n3 in (1 << 22, 1 << 23, 1 << 30):
        with pytest.raises(sm.SmapError) as e:
            sm.smap_plan(3, n3, 64, granularity="tile", persistent=8, device=sm.DEVICE_NONE)
        assert e.value.status == sm.E_INVALID and "64 bits" in str(e.value)
    q = sm.smap_plan_query(sm.smap_plan(3, 1 << 21, 64, granularity="tile", device=sm.DEVICE_NONE))
    assert q["useful_elems"] == math.comb(1 << 21, 3) and q["launched_threads"] == 3 * (1 << 21) ** 3 // 16
    plan3 = sm.smap_plan(3, 300, 8, map="below", granularity="tile", device=sm.DEVICE_NONE)
    with pytest.raises(sm.SmapError):
        sm.smap_locate(plan3, 3, 2, 1)                   # not i < j < k
