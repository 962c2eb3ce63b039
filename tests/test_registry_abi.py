"""Registry data and the C-ABI library surface (no GPU compute)."""

from __future__ import annotations

import ctypes
from ctypes import byref, c_double, c_int, c_int64

import pytest

from paper_1810_10496_b200 import _abi, registry
from paper_1810_10496_b200.irfeat import cosine_distance, extract_features, parse_ir


def test_descriptors_round_trip():
    for b in registry.BENCHES:
        for size, dims in registry.SIZES[b].items():
            text = registry.describe(b, dims)
            assert registry.parse_descriptor(text) == (b, tuple(dims))
    with pytest.raises(ValueError):
        registry.parse_descriptor("GEMM:ni=1")
    with pytest.raises(ValueError):
        registry.parse_descriptor("NOPE:n=1")


def test_ir_texts_parse_and_are_distinct_enough():
    feats = {b: extract_features(parse_ir(t)) for b, t in registry.IR_TEXTS.items()}
    assert all(f.norm() > 0 for f in feats.values())
    # contractions are each other's nearest neighbours; BLAS-2 likewise
    near = lambda q: min((cosine_distance(feats[q], feats[o]), o) for o in feats if o != q)[1]
    assert near("2MM") in ("3MM", "GEMM", "SYRK")
    assert near("ATAX") in ("BICG", "MVT")
    assert near("2DCONV") == "3DCONV"


def test_library_loads_and_exports_header_symbols():
    lib = _abi.lib()
    names = _abi.exported_symbols()
    assert len(names) >= 25
    for n in names:
        assert hasattr(lib, n), f"libpfgpu.so does not export {n}"
    assert lib.pf_abi_version() == 2
    assert lib.pf_bench_count() == 15


def test_variant_tables_and_registry_agree():
    lib = _abi.lib()
    for i, b in enumerate(registry.BENCHES):
        name = ctypes.create_string_buffer(32)
        nd, na = c_int(), c_int()
        _abi.check(lib.pf_bench_info(i, name, 32, byref(nd), byref(na)))
        assert name.value.decode() == b
        assert nd.value == len(registry.DIM_NAMES[b])
        for d in range(nd.value):
            buf = ctypes.create_string_buffer(16)
            _abi.check(lib.pf_bench_dim_name(i, d, buf, 16))
            assert buf.value.decode() == registry.DIM_NAMES[b][d]
        n = lib.pf_variant_count(i)
        assert n > 20
        knobs = (c_int * 5)()
        _abi.check(lib.pf_variant_knobs(i, 0, knobs))
        assert tuple(knobs) == (0, 0, 0, 0, 0)  # variant 0 is the baseline
        by, fl = c_double(), c_double()
        _abi.check(lib.pf_alg_work(i, _abi.dims_array(registry.SIZES[b]["config"]), byref(by), byref(fl)))
        assert by.value > 0 and fl.value > 0


def test_invalid_arguments_fail_loudly():
    lib = _abi.lib()
    assert lib.pf_bench_info(99, None, 0, None, None) == _abi.PF_EINVAL
    assert "range" in lib.pf_last_error().decode()
    knobs = (c_int * 5)()
    assert lib.pf_variant_knobs(0, 10_000, knobs) == _abi.PF_EINVAL


def test_artifacts_dedup_identical_sass():
    """Variants whose machine code is identical share an artifact digest."""
    from paper_1810_10496_b200.backend import b200

    for b in ("FDTD-2D", "2DCONV"):
        fam = b200.family(b)
        digests = {}
        for v in range(len(fam.knobs)):
            import hashlib

            digests.setdefault(hashlib.sha256(b200.variant_sass(b, v).encode()).hexdigest(), []).append(v)
        # knob-insensitive kernels (no loops) collapse
        assert len(digests) < len(fam.knobs)
