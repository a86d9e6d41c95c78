"""CPU-side checks of the C ABI: the library loads, exports every symbol include/oid.h declares,
validates parameters, and its Gauss-16 table equals the oracle's (built independently)."""

import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def oid():
    from __graft_entry__ import build
    build()
    import paper_2405_16076_b200 as oid
    return oid


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "oid.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(oid_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(oid):
    names = _declared_functions()
    assert len(names) >= 17
    lib = oid.lib()
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(oid.EXPORTED)


def test_version(oid):
    assert "sm_100a" in oid.version()


def test_sketch_table_matches_oracle(oid):
    from oracle import gauss16_levels, gauss16_scale
    q, s = oid.sketch_table()
    assert np.array_equal(q + 0.5, gauss16_levels())
    assert abs(s - gauss16_scale()) <= 2e-16 * s


def test_workspace_query_validates(oid):
    good = oid.make_params(m=4096, k=20, ell=48, b_max=16, n_cap=512, lam=1e-7, split=(16, 16, 16))
    assert oid.workspace_bytes(good) > 0
    bad_cases = [
        dict(m=4096, k=60, ell=48, b_max=16, n_cap=512, lam=0.0),                  # k > ell
        dict(m=4096, k=20, ell=48, b_max=65, n_cap=512, lam=0.0),                  # b_max > 64
        dict(m=4096, k=20, ell=48, b_max=16, n_cap=512, lam=-3.0),                 # bad lambda mode
        dict(m=4096, k=20, ell=48, b_max=16, n_cap=512, lam=0.0, split=(10, 10, 10)),
        dict(m=4096, k=20, ell=48, b_max=16, n_cap=512, lam=0.0, row_begin=100, row_end=50),
        dict(m=4096, k=20, ell=2000, b_max=16, n_cap=512, lam=0.0),                # ell > 1024
        dict(m=4096, k=20, ell=48, b_max=16, n_cap=512, lam=0.0, grad=(2, 32, 32)),  # 2*32*32 != m
        dict(m=4096, k=20, ell=700, b_max=16, n_cap=512, lam=0.0, grad=(4, 32, 32)),  # 3 ell > 2048
    ]
    # the gradient variant across row slabs is valid (halos through oid_ingest_sketch_halo)
    assert oid.workspace_bytes(oid.make_params(m=4096, k=20, ell=48, b_max=16, n_cap=512, lam=0.0, grad=(4, 32, 32),
                                               row_begin=0, row_end=2048)) > 0
    for kw in bad_cases:
        with pytest.raises(oid.OidError):
            oid.workspace_bytes(oid.make_params(**kw))


def test_struct_layout_matches_header(oid):
    # oid_params: 4 int64 + 6 int32 + 4 double + uint64 + 4 int32 = 32 + 24 + 32 + 8 + 16 = 112 bytes,
    # then the gradient-variant block: 4 int32 + 2 double = 32 bytes, then coeff_mode + epoch_mode,
    # then grad_nz + reserved1 + grad_hz (3-D gradients)
    assert ctypes.sizeof(oid.OidParams) == 168
    assert oid.OidParams.grad_nfields.offset == 112 and oid.OidParams.grad_hx.offset == 128
    assert oid.OidParams.coeff_mode.offset == 144
    # oid_stats_t: 4 int64 + 3 double + uint32 + int32, then a9_ms, 4 int64, 3 double
    assert ctypes.sizeof(oid.OidStats) == 4 * 8 + 3 * 8 + 8 + 8 + 4 * 8 + 3 * 8
    assert oid.OidStats.a9_ms.offset == 64 and oid.OidStats.lat_max_ms.offset == 120


def test_struct_layout_matches_compiled_header(oid, tmp_path):
    """The ctypes structs against the C compiler's view of include/oid.h (sizes and key offsets)."""
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "oid.h"\n'
                   'int main(void){printf("%zu %zu %zu %zu %zu\\n", sizeof(oid_params), offsetof(oid_params, coeff_mode),'
                   ' offsetof(oid_params, grad_hx), sizeof(oid_stats_t), offsetof(oid_stats_t, lat_max_ms)); return 0;}\n')
    exe = tmp_path / "sz"
    inc = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")
    subprocess.run(["gcc", "-I", inc, str(src), "-o", str(exe)], check=True)
    vals = [int(v) for v in subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()]
    assert vals == [ctypes.sizeof(oid.OidParams), oid.OidParams.coeff_mode.offset, oid.OidParams.grad_hx.offset,
                    ctypes.sizeof(oid.OidStats), oid.OidStats.lat_max_ms.offset]
