"""The C-ABI boundary: libenserve_b200.so loads, exports exactly what
include/enserve_b200.h declares, and maps the reference's error classes."""
from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2208_14049_b200 as es
from paper_2208_14049_b200 import _abi

HEADER = Path(__file__).resolve().parent.parent / "include" / "enserve_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^\s*(?:es_status|void|int|const char\*)\s+(es_\w+)\s*\(",
                                 text, flags=re.M)))


def test_library_exports_every_declared_symbol():
    names = declared_symbols()
    assert len(names) >= 40
    lib = ctypes.CDLL(str(es.LIB_PATH))
    for n in names:
        assert hasattr(lib, n), n
    assert sorted(_abi.EXPORTED) == names


def test_library_is_built_for_sm100a_with_tcgen05_and_tma():
    sass = subprocess.run(["cuobjdump", "-sass", str(es.LIB_PATH)], capture_output=True,
                          text=True).stdout
    if not sass:
        pytest.skip("cuobjdump unavailable")
    assert "UTCHMMA" in sass      # tcgen05.mma
    assert "UTMALDG" in sass      # TMA tile loads
    assert "LDTM" in sass         # tcgen05.ld (TMEM -> registers)
    elf = subprocess.run(["cuobjdump", "-lelf", str(es.LIB_PATH)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in elf


def test_abi_version_and_status_names():
    lib = es.lib()
    assert lib.es_abi_version() == es._abi.ABI_VERSION == 2
    assert lib.es_status_name(4) == b"ES_ERR_STARTUP"


def test_error_classes_cross_the_boundary():
    c = es.ClusterSpec([es.DeviceSpec(0, es.GPU, 1000.0, 1.0, 0.0)],
                       [es.ModelSpec(0, "oversized", 5000.0, 0.0, 1.0, 4)], [8], 128)
    with pytest.raises(es.AllocationError) as ei:
        es.worst_fit_decreasing(c, 8)
    assert ei.value.model_name == "oversized"
    with pytest.raises(es.SpecError):
        es.worst_fit_decreasing(c, 12)
    with pytest.raises(es.InvalidArgument):
        es.segment_bounds(3, 128, 300)
    with pytest.raises(es.BaselineError):
        es.bbs_baseline(es.ClusterSpec([es.DeviceSpec(0, es.GPU, 1e5, 1.0, 0.0)],
                                       [es.ModelSpec(0, "a", 1.0, 0.0, 1.0, 4),
                                        es.ModelSpec(1, "b", 1.0, 0.0, 1.0, 4)], [8], 128))


def test_product_does_not_link_the_oracle():
    deps = subprocess.run(["ldd", str(es.LIB_PATH)], capture_output=True, text=True).stdout
    assert "oracle" not in deps and "enserve_ref" not in deps
    import paper_2208_14049_b200.api as api
    src = Path(api.__file__).read_text() + Path(_abi.__file__).read_text()
    assert "oracle" not in src.replace("ORACLE", "")


def test_host_bf16_converter_rounds_to_nearest_even():
    from oracle.refcpu import round_bf16
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.standard_normal(100003).astype(np.float32) * 10,
                        np.array([0.0, -0.0, 1.0, 1.00390625, 1.0078125, 3.0e38, -3.0e-39],
                                 dtype=np.float32)])
    y = es.host_convert_bf16(x)
    want = (round_bf16(x).view(np.uint32) >> 16).astype(np.uint16)
    np.testing.assert_array_equal(y, want)


def test_host_bf16_converter_special_values_and_odd_lengths():
    # Inf keeps its sign, NaN stays a (quiet) NaN, on the vector and scalar paths alike
    for n in (7, 8, 33, 1000):
        x = np.linspace(-3, 3, n).astype(np.float32)
        x[n // 2] = np.inf
        x[0] = -np.inf
        x[-1] = np.nan
        y = es.host_convert_bf16(x)
        assert y[n // 2] == 0x7F80 and y[0] == 0xFF80
        assert (y[-1] & 0x7F80) == 0x7F80 and (y[-1] & 0x007F) != 0
        from oracle.refcpu import round_bf16
        finite = np.isfinite(x)
        want = (round_bf16(x[finite]).view(np.uint32) >> 16).astype(np.uint16)
        np.testing.assert_array_equal(y[finite], want)


def test_host_bf16_converter_keeps_subnormals_on_every_path():
    """fp32 subnormals become bf16 subnormals (RNE), as on the device, also
    inside the 32-wide vector loop (VCVTNE2PS2BF16 would flush them)."""
    from oracle.refcpu import round_bf16
    rng = np.random.default_rng(5)
    x = rng.standard_normal(4096).astype(np.float32)
    sub = (rng.random(4096) < 0.05)
    x[sub] = (rng.standard_normal(int(sub.sum())) * 1e-39).astype(np.float32)
    for off in (0, 1, 17):
        y = es.host_convert_bf16(x[off:])
        want = (round_bf16(x[off:]).view(np.uint32) >> 16).astype(np.uint16)
        np.testing.assert_array_equal(y, want)


def test_host_bf16_converter_concurrent_callers():
    """One process-wide pool, many Python threads (ctypes drops the GIL):
    every caller gets its whole array converted."""
    import threading
    from oracle.refcpu import round_bf16
    rng = np.random.default_rng(6)
    xs = [rng.standard_normal(200_000 + 37 * k).astype(np.float32) for k in range(8)]
    out = [None] * len(xs)

    def work(k):
        for _ in range(5):
            out[k] = es.host_convert_bf16(xs[k])

    ts = [threading.Thread(target=work, args=(k,)) for k in range(len(xs))]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    for k, x in enumerate(xs):
        want = (round_bf16(x).view(np.uint32) >> 16).astype(np.uint16)
        np.testing.assert_array_equal(out[k], want)
