"""The C-ABI libraries load and export every symbol their headers declare;
struct layouts of the ctypes mirror match the C compiler's; host-side
behaviour that needs no GPU."""
import ctypes as C
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from paper_1610_05108_b200 import _abi, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(xyzb_\w+)\s*\(", text)))


def test_libxyzb_exports_every_declared_symbol():
    lib = C.CDLL(_lib.LIB_PATH)
    names = declared("xyzb.h")
    assert "xyzb_search" in names and "xyzb_dataset_create" in names
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_abi.SIGNATURES), "ctypes mirror out of sync with include/xyzb.h"


def test_libxyzb_exports_the_test_hook():
    lib = C.CDLL(_lib.LIB_PATH)
    for name in declared("xyzb_testing.h"):
        assert hasattr(lib, name), name
    for name in _lib.TEST_OPTIONS:
        _lib.set_test_option(name, 0)  # known names; no device needed
    with pytest.raises(ValueError):
        _lib.set_test_option("no_such_option", 1)


def test_libxyzb_synth_exports_every_declared_symbol():
    lib = C.CDLL(_lib.SYNTH_PATH)
    for name in declared("xyzb_synth.h"):
        assert hasattr(lib, name), name


def test_abi_version_and_reference_defaults():
    lib = _lib.load()
    assert lib.xyzb_abi_version() == _abi.ABI_VERSION
    q = _abi.Params()
    lib.xyzb_params_init(C.byref(q))
    # SearchConfig defaults (search.hpp:18-33)
    assert (q.m, q.l, q.gamma, q.mode, q.transform, q.search_negatives, q.seed, q.max_candidates_per_rep,
            q.stop_after_first_hit, q.estimate_complexity, q.threads, q.strength_sample_size) == \
           (8, 1, 0.9, 0, 0, 1, 0, 0, 0, 1, 0, 0)


def test_struct_layouts_match_the_c_compiler():
    src = r"""
#include <stdio.h>
#include <stddef.h>
#include "xyzb.h"
#define F(T, m) printf(#T "." #m " %zu\n", offsetof(T, m));
int main(void) {
  printf("problem %zu\nresponse %zu\nparams %zu\nhit %zu\nresult %zu\n", sizeof(xyzb_problem),
         sizeof(xyzb_response), sizeof(xyzb_params), sizeof(xyzb_hit), sizeof(xyzb_result));
  F(xyzb_params, seed) F(xyzb_params, top_k) F(xyzb_params, rep_end)
  F(xyzb_hit, strength) F(xyzb_hit, sign)
  F(xyzb_result, stage_ms) F(xyzb_result, kernel_launches) F(xyzb_result, verify_launches)
  return 0;
}
"""
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "probe.c")
        open(c, "w").write(src)
        exe = os.path.join(d, "probe")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", exe, c])
        out = dict(line.rsplit(" ", 1) for line in subprocess.check_output([exe]).decode().split("\n") if line)
    assert int(out["problem"]) == C.sizeof(_abi.Problem)
    assert int(out["response"]) == C.sizeof(_abi.Response)
    assert int(out["params"]) == C.sizeof(_abi.Params)
    assert int(out["hit"]) == C.sizeof(_abi.Hit)
    assert int(out["result"]) == C.sizeof(_abi.Result)
    assert int(out["xyzb_params.seed"]) == _abi.Params.seed.offset
    assert int(out["xyzb_params.top_k"]) == _abi.Params.top_k.offset
    assert int(out["xyzb_params.rep_end"]) == _abi.Params.rep_end.offset
    assert int(out["xyzb_hit.strength"]) == _abi.Hit.strength.offset
    assert int(out["xyzb_hit.sign"]) == _abi.Hit.sign.offset
    assert int(out["xyzb_result.stage_ms"]) == _abi.Result.stage_ms.offset
    assert int(out["xyzb_result.kernel_launches"]) == _abi.Result.kernel_launches.offset
    assert int(out["xyzb_result.verify_launches"]) == _abi.Result.verify_launches.offset


def _has_gpu():
    try:
        return _lib.load().xyzb_device_count() > 0
    except Exception:
        return False


@pytest.mark.skipif(_has_gpu(), reason="checks the no-device behaviour")
def test_no_cpu_fallback_without_a_device():
    import paper_1610_05108_b200 as xb
    x = xb.PackedMatrix.from_signs(np.ones((10, 3), np.int8))
    with pytest.raises(xb.CudaError):
        xb.Dataset(x)


def test_dataset_create_validates_before_device_work():
    import paper_1610_05108_b200 as xb
    x = xb.PackedMatrix(70, 2)
    x.words[1, 1] = np.uint64(1) << np.uint64(63)  # padding bit set
    with pytest.raises(xb.DataError):
        xb.Dataset(x)


def test_packing_roundtrip_and_pack_signs():
    import paper_1610_05108_b200 as xb
    rng = np.random.default_rng(0)
    for n in (1, 63, 64, 65, 200):
        s = np.where(rng.random((n, 7)) < 0.5, 1, -1).astype(np.int8)
        x = xb.PackedMatrix.from_signs(s)
        assert x.padding_clear()
        assert np.array_equal(x.to_signs(), s)
        assert all(x.get(i, j) == s[i, j] for i in range(n) for j in range(7))
        y = s[:, 0]
        yw = xb.pack_signs(y)
        assert all(((int(yw[i >> 6]) >> (i & 63)) & 1) == (y[i] > 0) for i in range(n))


def test_synthetic_toy_is_the_reference_recipe():
    from paper_1610_05108_b200 import synth
    from tests import checkers as ck
    if not ck.ref_available():
        pytest.skip("oracle/_ref not built")
    x, y = synth.toy()
    xr, yr = ck.ref_planted(1000, 2000, 4, 16, 0.9, 1)
    assert np.array_equal(x.words, xr.words) and np.array_equal(y, yr)
