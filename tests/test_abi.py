"""CPU-side checks of the C ABI boundary (no compute calls; no GPU needed).

The library loads, exports every function include/alp.h declares, its struct layouts match
ctypes (checked against a gcc-compiled probe of the header), its default constants equal the
oracle's, and argument validation fails synchronously with the documented
status codes before any CUDA call.
"""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "alp.h")


@pytest.fixture(scope="module")
def lib():
    from paper_0902_0657_b200 import build, _ffi
    build.build()
    return _ffi.load()


def header_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^[A-Za-z_][\w \*]*?\b([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)))


def test_exports_every_declared_symbol(lib):
    names = header_functions()
    assert {"alp_decode", "ipm_step_pcg", "alp_code_create", "alp_decode_host"} <= set(names)
    so = os.path.join(ROOT, "paper_0902_0657_b200", "libalp.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(line.split()[-1] for line in out.splitlines() if line.strip())
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    for n in names:
        getattr(lib, n)


def test_struct_layout_matches_header(lib):
    from paper_0902_0657_b200._ffi import AlpParams, FrameStats
    probe = r"""
#include <stdio.h>
#include <stddef.h>
#include "alp.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu\n", sizeof(alp_params), offsetof(alp_params, sigma),
         offsetof(alp_params, alp_max_iter), offsetof(alp_params, warps_per_block),
         sizeof(alp_frame_stats));
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        cpath = os.path.join(d, "probe.c")
        open(cpath, "w").write(probe)
        exe = os.path.join(d, "probe")
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), cpath, "-o", exe], check=True)
        vals = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    assert vals == [C.sizeof(AlpParams), AlpParams.sigma.offset, AlpParams.alp_max_iter.offset,
                    AlpParams.warps_per_block.offset, C.sizeof(FrameStats)]
    assert C.sizeof(FrameStats) == 128


def test_default_params_equal_oracle_constants(lib):
    from paper_0902_0657_b200 import default_params
    from oracle.lp import DEFAULT_PARAMS
    p = default_params()
    for k, v in DEFAULT_PARAMS.items():
        assert getattr(p, k) == v, k
    assert p.variant == 0 and p.precond == 0


def _create(lib, n, m, rp, ci):
    h = C.c_void_p()
    rp = np.ascontiguousarray(rp, dtype=np.int32)
    ci = np.ascontiguousarray(ci, dtype=np.int32)
    st = lib.alp_code_create(n, m, rp.ctypes.data, ci.ctypes.data, C.byref(h))
    return st, h


def test_code_validation_is_synchronous(lib):
    assert _create(lib, 4, 2, [0, 3, 6], [0, 1, 4, 1, 2, 3])[0] == -2        # out of range
    assert _create(lib, 4, 2, [0, 3, 6], [0, 2, 1, 1, 2, 3])[0] == -2        # not increasing
    assert _create(lib, 4, 2, [0, 3, 3], [0, 1, 2])[0] == -2                 # empty check
    assert _create(lib, 4, 2, [1, 3, 6], [0, 1, 2, 1, 2, 3])[0] == -2        # row_ptr[0] != 0
    assert _create(lib, 0, 2, [0, 3, 6], [0, 1, 2, 1, 2, 3])[0] == -1        # n <= 0
    n = 20
    assert _create(lib, n, 1, [0, 16], list(range(16)))[0] == -3             # d_c > 15
    rows = [[0, j + 1] for j in range(5)]                                    # var 0 has degree 5
    rp = np.cumsum([0] + [len(r) for r in rows])
    assert _create(lib, 6, 5, rp, sum(rows, []))[0] == -3
    assert b"variable degree" in lib.alp_last_error()
    assert lib.alp_status_string(-5) == b"ALP_ERR_WORKSPACE"


def test_null_arguments_rejected(lib):
    from paper_0902_0657_b200._ffi import AlpParams
    assert lib.alp_decode(None, 1, None, None, None, None, None, None, None, None, None, None, 0,
                          None, None) == -1
    assert lib.ipm_step_pcg(None, 1, None, None, None, None, None, None, None, None, None, None,
                            None, 0, None, None) == -1
    p = AlpParams()
    lib.alp_default_params(C.byref(p))
    p.variant = 7
    assert lib.alp_decode(None, 1, None, None, None, None, None, None, None, None, None, None, 0,
                          C.byref(p), None) == -1


def test_product_package_does_not_import_oracle():
    import paper_0902_0657_b200
    pkg = os.path.dirname(paper_0902_0657_b200.__file__)
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", src, flags=re.M), fn
