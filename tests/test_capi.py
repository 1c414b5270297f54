"""The C-ABI library on CPU: it loads, exports every symbol include/fier_cuda.h
declares, and its host-only logic (FIER format conversion, argument validation
with the reference's error texts) behaves like the reference.  No kernel is
launched here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_cases, load_golden

HEADER = os.path.join(ROOT, "include", "fier_cuda.h")


@pytest.fixture(scope="module")
def lib():
    from paper_2508_08256_b200 import _lib
    return _lib.load()


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*FIER_API\s+(?:const\s+)?\w+\*?\s+\**(fier_\w+)\(", text, re.M)))


def test_exports_every_declared_symbol(lib):
    from paper_2508_08256_b200 import _lib
    names = header_functions()
    assert len(names) >= 19
    assert set(names) == set(_lib.EXPORTS)
    for name in names:
        assert hasattr(lib, name), name


def test_library_is_sm100a(lib):
    from paper_2508_08256_b200 import _lib
    blob = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in blob


def test_payload_bytes_match_reference_accounting(lib):
    # PackedKeys::payload_bytes (quant1bit.hpp:60-62), acceptance_main.cpp:66-109
    assert lib.fier_payload_bytes(4096, 128, 32) == 4096 * 128 // 8 + (4096 * 128 // 32) * 4
    assert lib.fier_payload_bytes(100, 11, 32) == 100 * 2 + 11 * 4 * 4
    assert lib.fier_payload_bytes(0, 11, 32) == 0


@pytest.mark.parametrize("name", golden_cases())
def test_fier_format_round_trip(lib, name):
    """Host conversion device-layout <-> FIER bytes is exact on reference fixtures."""
    c = load_golden(name)
    for buf in c["fier_list"]:
        b = np.frombuffer(buf, np.uint8)
        l, d, g = C.c_int32(), C.c_int32(), C.c_int32()
        assert lib.fier_fier_to_index(b.ctypes.data, b.size, C.byref(l), C.byref(d), C.byref(g),
                                      None, 0, None, 0) == 0
        assert (l.value, d.value, g.value) == (c["l"], c["d"], c["g"])
        W = (c["d"] + 31) // 32
        G = (c["l"] + c["g"] - 1) // c["g"]
        bits = np.zeros(c["l"] * W, np.uint32)
        par = np.zeros(G * c["d"] * 2, np.uint16)
        assert lib.fier_fier_to_index(b.ctypes.data, b.size, C.byref(l), C.byref(d), C.byref(g),
                                      bits.ctypes.data, bits.size, par.ctypes.data, par.size) == 0
        out = np.zeros(len(buf), np.uint8)
        assert lib.fier_index_to_fier(bits.ctypes.data, par.ctypes.data, l, d, g, out.ctypes.data,
                                      out.size) == 0
        assert out.tobytes() == buf


def test_fier_parse_diagnostics(lib):
    """Rejections name the violated field like parse_packed_keys (test_io.cpp:169-190)."""
    from paper_2508_08256_b200 import _lib
    c = load_golden("short_group_d24")
    good = c["fier_list"][0]

    def parse(buf):
        b = np.frombuffer(buf, np.uint8)
        l, d, g = C.c_int32(), C.c_int32(), C.c_int32()
        rc = lib.fier_fier_to_index(b.ctypes.data, b.size, C.byref(l), C.byref(d), C.byref(g),
                                    None, 0, None, 0)
        return rc, _lib.last_error()

    bad = bytearray(good)
    bad[1] = ord("?")
    assert parse(bytes(bad)) == (2, "bad magic: expected FIER")
    assert parse(good[:-1])[0] == 2 and "payload length mismatch" in parse(good[:-1])[1]
    bad = bytearray(good)
    bad[14:18] = b"\0\0\0\0"
    assert parse(bytes(bad)) == (2, "invalid g: must be >= 1")
    bad = bytearray(good)
    bad[4] = 9
    assert parse(bytes(bad)) == (2, "unsupported version: 9")


def test_validation_uses_reference_messages(lib):
    """Precondition failures return FIER_EINVAL before any launch (no GPU needed)."""
    from paper_2508_08256_b200 import _lib
    from paper_2508_08256_b200.api import make_shape
    s = make_shape(1, 2, 2, 64, 128, 32, _lib.FIER_BF16)
    dummy = C.c_void_p(16)
    assert lib.fier_topk(dummy, 1, 10, 10, 0, dummy, None, 0, None) == 1
    assert _lib.last_error() == "topk_oracle: k out of range"
    assert lib.fier_topk(dummy, 1, 10, 10, 11, dummy, None, 0, None) == 1
    assert lib.fier_sparse_attention(C.byref(s), dummy, dummy, dummy, dummy, 0, 10, 1.0, dummy,
                                     dummy, 1 << 20, None) == 1
    assert _lib.last_error() == "gather_attention: empty selection"
    assert lib.fier_sparse_attention(C.byref(s), dummy, dummy, dummy, dummy, 11, 10, 1.0, dummy,
                                     dummy, 1 << 20, None) == 1
    assert _lib.last_error() == "gather_attention: selection invalid for cache"
    assert lib.fier_decode_step(C.byref(s), dummy, dummy, dummy, 9, dummy, dummy, dummy, dummy, 11,
                                1.0, dummy, dummy, None, dummy, 1 << 30, None) == 1
    assert _lib.last_error() == "fier_select: budget out of range"
    bad_g = make_shape(1, 2, 2, 64, 128, 0, _lib.FIER_BF16)
    assert lib.fier_pack_keys(C.byref(bad_g), dummy, 10, dummy, dummy, None, None) == 1
    assert _lib.last_error() == "quantize: group size must be >= 1"
    assert lib.fier_pack_keys(C.byref(s), dummy, 0, dummy, dummy, None, None) == 1
    assert _lib.last_error() == "quantize: empty key cache"
    gqa_bad = make_shape(1, 3, 2, 64, 128, 32, _lib.FIER_BF16)
    assert lib.fier_score(C.byref(gqa_bad), dummy, dummy, dummy, 10, dummy, 10, None) == 1


def test_python_api_raises_value_error_like_reference():
    from paper_2508_08256_b200 import _lib
    with pytest.raises(ValueError, match="topk_oracle: k out of range"):
        _lib.check(_lib.load().fier_topk(C.c_void_p(16), 1, 4, 4, 5, C.c_void_p(16), None, 0, None))


def test_workspace_sizes_are_consistent(lib):
    from paper_2508_08256_b200 import _lib
    from paper_2508_08256_b200.api import make_shape
    s = make_shape(1, 32, 32, 32768, 128, 32, _lib.FIER_BF16)
    assert lib.fier_bits_bytes(C.byref(s)) == 32 * 32768 * 16
    assert lib.fier_params_bytes(C.byref(s)) == 32 * 1024 * 128 * 4
    ws = lib.fier_decode_workspace(C.byref(s), 32768, 3604)
    assert ws >= 32 * 32768 * 4
    assert lib.fier_step_scores_ld(33) == 64


def test_sass_has_no_odd_memory_descriptor_registers():
    """Regression guard: ptxas 12.9 once emitted LDGSTS with desc[UR1] (odd uniform
    register as a 64-bit descriptor), which traps as an illegal instruction on B200."""
    import shutil
    import subprocess
    from paper_2508_08256_b200 import _lib
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    sass = subprocess.run([tool, "-sass", _lib.LIB_PATH], capture_output=True, text=True, check=True).stdout
    assert "LDGSTS" in sass
    assert not re.search(r"desc\[UR\d*[13579]\]", sass)


def _read_blobs(path):
    out = []
    with open(path, "rb") as f:
        data = f.read()
    off = 0
    dtypes = [np.float64, np.float64, np.float64, np.uint64, np.float64, np.float64, np.float64, np.int64,
              np.float64, np.int64, np.float64, np.uint8, np.uint8,
              np.float64, np.float64, np.float64, np.int64, np.int64]  # + Quest: K, kmax, kmin, sel, sel_q
    for dt in dtypes:
        n = int(np.frombuffer(data[off:off + 8], np.uint64)[0])
        off += 8
        nbytes = n * np.dtype(dt).itemsize
        out.append(np.frombuffer(data[off:off + nbytes], dt).copy())
        off += nbytes
    return out


@pytest.mark.gpu
def test_cpp_shim_matches_oracle(cuda, port, tmp_path):
    """Host C++ through include/fier_cuda.hpp (fier::cuda::quantize / approx_scores /
    topk_oracle / gather_attention / fier_select / fier_attend / build_page_summaries /
    quest_select / quest_select_quantized) against the oracle."""
    import subprocess
    from paper_2508_08256_b200 import build as b
    exe = b.SHIM_BIN
    if not os.path.exists(exe):
        exe = b.build_shim_test()
    res = str(tmp_path / "shim.bin")
    r = subprocess.run([exe, res], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    K, V, q, cw, s, z, est, sel, out, sel2, out2, e1, e2, KQ, qmax, qmin, qs, qq = _read_blobs(res)
    l, d, g, n = 1000, 128, 32, 77
    K, V = K.reshape(l, d), V.reshape(l, d)
    cw_ref, s_ref, z_ref = port.quantize(K, g)
    assert np.array_equal(cw, cw_ref)  # bit-exact code words
    rh = np.vectorize(lambda x: port.half_to_double(port.double_to_half(x)))
    assert np.array_equal(s, rh(s_ref)) and np.array_equal(z, rh(z_ref))  # == round_through_half
    buf = port.serialize(l, d, g, cw, s, z)
    assert buf == port.quantize_fier(K, g)  # serialize_packed_keys byte-identical
    ref_scores = port.approx_scores_fier(q, buf)
    assert np.max(np.abs(est - ref_scores) / np.maximum(1, np.abs(ref_scores))) <= 1e-3
    assert np.array_equal(sel, port.topk(est, n))
    assert np.array_equal(sel2, sel)
    want = port.gather_attention(q, K, V, sel)
    assert port.relative_l2_error(out, want) < 1e-2
    assert port.relative_l2_error(out2, want) < 1e-2
    assert bytes(e1).decode() == "topk_oracle: k out of range"
    assert bytes(e2).decode() == "fier_select: budget out of range"
    # Quest through the shim (baselines.hpp): exact summaries, the oracle's selections
    KQ = KQ.reshape(4096, d)
    kmax, kmin = port.page_summaries(KQ, 16)
    assert np.array_equal(qmax.reshape(kmax.shape), kmax) and np.array_equal(qmin.reshape(kmin.shape), kmin)
    assert np.array_equal(qs, port.quest_select(q, KQ, 16, 300, "sum"))
    bufq = port.quantize_fier(KQ, g)
    est_q = port.approx_scores_fier(q, bufq)
    assert np.array_equal(qq, port.select_by_page_scores(port.page_mean(est_q, 16), 4096, 16, 300))


@pytest.mark.parametrize("l,g", [(4096, 32), (4096, 128), (4096, 256), (4096, 1), (100, 32), (1, 1), (33, 32),
                                 (131072, 32), (1048577, 32), (7, 1000)])
def test_load_ratio_fier_matches_reference(l, g):
    """fier_load_ratio_fier == the reference's load_ratio_fier (quant1bit.hpp:176-184) on exact
    bit counts, the reduced Rational and the formula flag (acceptance_main.cpp:66-109: 0.125,
    0.078125, 0.0703125 at g = 32, 128, 256; short groups force exact accounting)."""
    import paper_2508_08256_b200 as F
    from oracle.oracle import Ref, REF_SO
    r = F.load_ratio_fier(l, g)
    if os.path.exists(REF_SO):
        bits, ratio, formula = Ref().load_ratio_fier(l, g)
        assert (r.numerator_bits, r.denominator_bits) == bits
        assert r.ratio() == ratio and r.formula == formula
    expect = {(4096, 32): 0.125, (4096, 128): 0.078125, (4096, 256): 0.0703125}
    if (l, g) in expect:
        assert r.value() == expect[(l, g)] and r.formula
    with pytest.raises(ValueError, match="load_ratio_fier: l and g must be >= 1"):
        F.load_ratio_fier(0, g)


def test_nccl_exchange_library_exports_its_header():
    """libfier_nccl.so (the NCCL device-API exchange, include/fier_nccl.h) loads without a GPU
    and exports every declared function; built by __graft_entry__.build() where torch's NCCL
    ships the device-API headers."""
    import ctypes
    import re
    from paper_2508_08256_b200 import build as b
    path = b.build_nccl()
    if not path:
        pytest.skip("no NCCL with the device API in this environment")
    lib = ctypes.CDLL(path)
    text = open(os.path.join(ROOT, "include", "fier_nccl.h")).read()
    names = re.findall(r"FIER_API\s+[\w\s\*]+?\b(fier_devx_\w+)\s*\(", text)
    assert len(names) == 6
    for name in names:
        assert hasattr(lib, name), name
    assert b"sm_100a" in open(path, "rb").read()
