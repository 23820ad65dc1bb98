"""C-ABI library checks that need no GPU: it loads, exports every symbol that
include/bitserial.h declares, and rejects bad arguments before touching CUDA."""
import ctypes
import os
import re

import pytest

import paper_1810_11066_b200 as bs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "bitserial.h")


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(bs.library_path()):
        from paper_1810_11066_b200 import build
        build.build()
    return bs._load()


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bs_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("bs_bitpack", "bs_bitserial_dense", "bs_bitserial_conv2d_nhwc"):
        assert required in names
    assert set(names) == set(bs.EXPORTED_SYMBOLS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_exports_are_c_symbols():
    out = os.popen(f"nm -D --defined-only {bs.library_path()}").read()
    exported = set(re.findall(r"\bT (bs_[a-z0-9_]+)\b", out))
    assert set(declared_functions()) <= exported


def test_abi_version_and_row_words(lib):
    import oracle
    assert bs.abi_version() == 1
    for k in (1, 31, 32, 33, 64, 65, 100, 576, 4096, 4097):
        assert bs.packed_row_words(k) == oracle.packed_row_words(k)
    assert bs.packed_row_words(0) == 0


def test_status_strings(lib):
    assert lib.bs_status_string(0) == b"BS_OK"
    assert lib.bs_status_string(4) == b"BS_ERR_SHAPE"
    assert lib.bs_status_string(99) == b"BS_ERR_UNKNOWN"


NULL = ctypes.c_void_p(0)
FAKE = ctypes.c_void_p(0x10000)       # never dereferenced: validation fails first
MISALIGNED = ctypes.c_void_p(0x10004)


def test_validation_before_launch(lib):
    # null pointers
    assert lib.bs_bitpack(NULL, FAKE, 4, 32, 2, NULL) == 1
    assert lib.bs_bitserial_dense(FAKE, 2, NULL, 1, 1, FAKE, 1, 1, 1, NULL) == 1
    # bits out of range / bad encoding / bad algo
    assert lib.bs_bitpack(FAKE, FAKE, 4, 32, 9, NULL) == 2
    assert lib.bs_bitserial_dense(FAKE, 0, FAKE, 1, 1, FAKE, 1, 1, 1, NULL) == 2
    assert lib.bs_bitserial_dense(FAKE, 2, FAKE, 1, 7, FAKE, 1, 1, 1, NULL) == 2
    assert lib.bs_bitserial_dense_ex(FAKE, 2, FAKE, 1, 1, FAKE, 1, 1, 1, 42, NULL) == 2
    # shapes
    assert lib.bs_bitpack(FAKE, FAKE, 0, 32, 2, NULL) == 4
    assert lib.bs_bitserial_dense(FAKE, 2, FAKE, 1, 1, FAKE, 1, 0, 1, NULL) == 4
    # empty conv output: 3x3 kernel on 2x2 input, no pad
    assert lib.bs_bitserial_conv2d_nhwc(FAKE, 2, FAKE, 1, 1, FAKE, 1, 2, 2, 8, 4, 3, 3, 1, 1, 0, 0, NULL) == 4
    # stride / pad
    assert lib.bs_bitserial_conv2d_nhwc(FAKE, 2, FAKE, 1, 1, FAKE, 1, 8, 8, 8, 4, 3, 3, 0, 1, 1, 1, NULL) == 2
    assert lib.bs_bitserial_conv2d_nhwc(FAKE, 2, FAKE, 1, 1, FAKE, 1, 8, 8, 8, 4, 3, 3, 1, 1, -1, 1, NULL) == 2
    # alignment
    assert lib.bs_bitpack(MISALIGNED, FAKE, 4, 32, 2, NULL) == 5
    # accumulator bound: K (2^8-1)^2 >= 2^31
    assert lib.bs_bitserial_dense(FAKE, 8, FAKE, 8, 0, FAKE, 1, 1, 40000, NULL) == 6
    # workspace too small
    assert lib.bs_bitserial_conv2d_nhwc_i8(FAKE, 2, FAKE, 1, 1, FAKE, 1, 8, 8, 64, 4, 3, 3, 1, 1, 1, 1,
                                           FAKE, 16, NULL) == 8
    assert b"workspace" in lib.bs_last_error()


def test_output_row_bound(lib):
    """Launches index output rows (M) in 32 bits: shapes past 2^31 - 257 rows are refused
    before launch (BS_ERR_SHAPE), including a conv whose padding makes the output larger
    than its input (n*h*w < 2^31 but n*oh*ow > 2^31; 3x3, pad 2 -> oh = h + 2)."""
    n, h = 131072, 127
    assert n * h * h < 2 ** 31 - 1 and n * (h + 2) * (h + 2) > 2 ** 31 - 257
    assert lib.bs_bitserial_conv2d_nhwc(FAKE, 2, FAKE, 1, 1, FAKE, n, h, h, 32, 4, 3, 3, 1, 1, 2, 2, NULL) == 4
    assert b"output pixels" in lib.bs_last_error()
    # dense: m past the row bound; n past 2^31 - 1 on the tile kernels (m > 8; the GEMV for
    # m <= 8 indexes n in 64 bits and takes it)
    assert lib.bs_bitserial_dense(FAKE, 2, FAKE, 1, 1, FAKE, 2 ** 31 - 1, 8, 64, NULL) == 4
    assert lib.bs_bitserial_dense(FAKE, 2, FAKE, 1, 1, FAKE, 16, 2 ** 31, 64, NULL) == 4
    assert b"m or n too large" in lib.bs_last_error()


def test_gemv_algo_rejected_for_conv(lib):
    assert lib.bs_bitserial_conv2d_nhwc_ex(FAKE, 2, FAKE, 1, 1, FAKE, 1, 8, 8, 8, 4, 3, 3, 1, 1, 1, 1, 3, NULL) == 3


def test_binding_refuses_cpu_tensors():
    import torch
    with pytest.raises(bs.BitserialError):
        bs.bitpack(torch.zeros(4, 32, dtype=torch.uint8), 2)


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_1810_11066_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liboracle" not in text and "oracle.c" not in text, f


def test_tc_validation_before_launch(lib):
    # bad tensor-core format
    assert lib.bs_bitserial_dense_tc_prepared(FAKE, 2, 0, FAKE, 1, 0, 7, FAKE, 16, 16, 64, NULL) == 2
    # FP4 format exactness bound: K (2^4-1)(2^2-1) = 45 K >= 2^22 for K = 100000 (I8 accepts it)
    assert lib.bs_bitserial_dense_tc_prepared(FAKE, 4, 0, FAKE, 2, 0, bs.TC_F4, FAKE, 16, 16, 100000, NULL) == 6
    assert b"2^22" in lib.bs_last_error()
    # unsupported precision for the tensor-core path (A in [1,4], W in [1,2])
    assert lib.bs_bitserial_dense_tc_prepared(FAKE, 5, 0, FAKE, 1, 0, bs.TC_I8, FAKE, 16, 16, 64, NULL) == 3
    # encodings: bad a_enc; bipolar / signed activations need the FP4 format
    assert lib.bs_bitserial_dense_tc_prepared(FAKE, 2, 3, FAKE, 1, 0, bs.TC_F4, FAKE, 16, 16, 64, NULL) == 2
    assert lib.bs_bitserial_dense_tc_prepared(FAKE, 2, 1, FAKE, 1, 1, bs.TC_I8, FAKE, 16, 16, 64, NULL) == 3
    assert lib.bs_dense_tc_prepare_weights(FAKE, 1, 3, 64, 64, bs.TC_F4, FAKE, 1 << 20, NULL) == 2
    # prepared-weight buffer too small
    assert lib.bs_dense_tc_prepare_weights(FAKE, 1, 1, 64, 64, bs.TC_F4, FAKE, 16, NULL) == 8
    # weight bytes per format: I8 32 B per packed word and plane, K words padded to 4; F4 16 B
    # per packed word and radix-4 digit (ceil(W/2) digits), K words padded to 8 (256-element
    # chunks); K = 64 -> 2 words
    assert lib.bs_dense_tc_weight_bytes(64, 64, 1, bs.TC_I8) == 64 * 4 * 32
    assert lib.bs_dense_tc_weight_bytes(64, 64, 2, bs.TC_I8) == 2 * 64 * 4 * 32
    assert lib.bs_dense_tc_weight_bytes(64, 64, 2, bs.TC_F4) == 1 * 64 * 8 * 16
    assert lib.bs_dense_tc_weight_bytes(64, 64, 3, bs.TC_F4) == 2 * 64 * 8 * 16
    assert lib.bs_dense_tc_weight_bytes(64, 300, 1, bs.TC_F4) == 1 * 64 * 16 * 16  # 10 words -> 16
    assert lib.bs_dense_tc_weight_bytes(64, 64, 1, 9) == 0


def _desc(**kw):
    d = bs.TcConvDesc()
    d.act_packed = d.w_tc = d.out = 1 << 20  # fake, 16-byte aligned device pointers (never dereferenced)
    d.n, d.h, d.w, d.c, d.oc, d.kh, d.kw, d.stride_h, d.stride_w, d.pad_h, d.pad_w = 1, 8, 8, 64, 64, 3, 3, 1, 1, 1, 1
    for k, v in kw.items():
        setattr(d, k, v)
    return d


def test_tc_group_validation_before_launch(lib):
    """bs_bitserial_conv2d_nhwc_tc_group validates every descriptor before launching
    anything (no GPU here: a launch would fail with a CUDA error, not these codes)."""
    import ctypes
    arr = (bs.TcConvDesc * 3)(_desc(), _desc(oc=0), _desc())
    p = ctypes.cast(arr, ctypes.c_void_p)
    assert lib.bs_bitserial_conv2d_nhwc_tc_group(p, 0, 2, 1, bs.TC_F4, NULL) == 0  # empty: no-op
    assert lib.bs_bitserial_conv2d_nhwc_tc_group(NULL, 2, 2, 1, bs.TC_F4, NULL) == 1  # NULL array
    assert lib.bs_bitserial_conv2d_nhwc_tc_group(p, 3, 2, 1, bs.TC_F4, NULL) == 4  # member 1: oc = 0
    arr[1] = _desc(out=0)
    assert lib.bs_bitserial_conv2d_nhwc_tc_group(p, 3, 2, 1, bs.TC_F4, NULL) == 1  # NULL out
    arr[1] = _desc(w_tc=(1 << 20) + 4)
    assert lib.bs_bitserial_conv2d_nhwc_tc_group(p, 3, 2, 1, bs.TC_F4, NULL) == 5  # misaligned
    arr[1] = _desc(a_enc=bs.A_BIPOLAR)
    assert lib.bs_bitserial_conv2d_nhwc_tc_group(p, 3, 2, 1, bs.TC_I8, NULL) == 3  # bipolar A needs FP4
    assert lib.bs_bitserial_conv2d_nhwc_tc_group(p, 3, 5, 1, bs.TC_F4, NULL) == 3  # A5 unsupported
    assert lib.bs_bitserial_conv2d_nhwc_tc_group(p, 3, 2, 1, 7, NULL) == 2  # bad format
    arr[1] = _desc(c=100000, kh=1, kw=1, pad_h=0, pad_w=0)
    assert lib.bs_bitserial_conv2d_nhwc_tc_group(p, 3, 4, 2, bs.TC_F4, NULL) == 6  # FP4 bound 2^22


def test_bitpack_group_validation(lib):
    import ctypes
    arr = (bs.PackDesc * 2)()
    for d in arr:
        d.in_, d.out, d.rows, d.k = 1 << 20, 1 << 21, 10, 64
    p = ctypes.cast(arr, ctypes.c_void_p)
    assert lib.bs_bitpack_group(p, 0, 2, NULL) == 0
    assert lib.bs_bitpack_group(NULL, 2, 2, NULL) == 1
    assert lib.bs_bitpack_group(p, 2, 9, NULL) == 2
    arr[1].k = 0
    assert lib.bs_bitpack_group(p, 2, 2, NULL) == 4
    arr[1].k, arr[1].out = 64, (1 << 21) + 4
    assert lib.bs_bitpack_group(p, 2, 2, NULL) == 5


def test_dense_gather_validation(lib):
    import ctypes
    peers = (ctypes.c_void_p * 9)(*([1 << 20] * 9))
    pp = ctypes.cast(peers, ctypes.c_void_p)
    f = lib.bs_bitserial_dense_tc_prepared_gather
    assert f(FAKE, 2, 0, FAKE, 1, 1, bs.TC_F4, FAKE, pp, 9, 16, 16, 64, NULL) == 2   # npeers > 8
    assert f(FAKE, 2, 0, FAKE, 1, 1, bs.TC_F4, FAKE, NULL, 2, 16, 16, 64, NULL) == 1  # NULL peer list
    assert f(FAKE, 2, 0, FAKE, 1, 1, bs.TC_F4, FAKE, pp, 2, 16, 18, 64, NULL) == 3   # n % 4 != 0
    peers[1] = (1 << 20) + 4
    assert f(FAKE, 2, 0, FAKE, 1, 1, bs.TC_F4, FAKE, pp, 2, 16, 16, 64, NULL) == 5   # misaligned peer
    peers[1] = 0
    assert f(FAKE, 2, 0, FAKE, 1, 1, bs.TC_F4, FAKE, pp, 2, 16, 16, 64, NULL) == 1   # NULL peer


def test_tc_host_group_validation(lib):
    import ctypes
    d = (bs.TcHostDesc * 1)()
    x = d[0]
    x.act_host = x.out_host = 1 << 20
    x.act_dev = x.packed_dev = x.out_dev = x.w_tc = 1 << 21
    x.n, x.h, x.w, x.c, x.oc, x.kh, x.kw, x.stride_h, x.stride_w, x.pad_h, x.pad_w = 1, 8, 8, 64, 64, 3, 3, 1, 1, 1, 1
    p = ctypes.cast(d, ctypes.c_void_p)
    f = lib.bs_bitserial_conv2d_nhwc_tc_host_group
    assert f(p, 0, 2, 1, bs.TC_F4, NULL) == 0
    assert f(NULL, 1, 2, 1, bs.TC_F4, NULL) == 1
    assert f(p, 1, 2, 1, 7, NULL) == 2
    x.out_dev = 0
    assert f(p, 1, 2, 1, bs.TC_F4, NULL) == 1
    x.out_dev = (1 << 21) + 8
    assert f(p, 1, 2, 1, bs.TC_F4, NULL) == 5
    x.out_dev, x.oc = 1 << 21, 0
    assert f(p, 1, 2, 1, bs.TC_F4, NULL) == 4


@pytest.mark.parametrize("geom", [
    (256, 56, 56, 64, 3, 3, 1, 1), (256, 56, 56, 64, 3, 3, 2, 1), (256, 56, 56, 64, 1, 1, 2, 0),
    (256, 7, 7, 512, 3, 3, 1, 1), (2, 5, 4, 40, 3, 3, 1, 1), (1, 6, 7, 33, 3, 3, 2, 1), (1, 5, 6, 20, 2, 3, 1, 0),
    (1, 7, 5, 96, 3, 2, 2, 2), (4, 11, 11, 3, 5, 3, 1, 2), (1, 5, 6, 64, 7, 7, 1, 3)])
@pytest.mark.parametrize("bits", [1, 2, 3, 4])
def test_tcw_layout_size_matches_the_oracle_definition(lib, geom, bits):
    """The library's window-layout size (host code, no GPU) equals the size the oracle's
    definition of the layout (R26) gives: ceil(bits/2) x phases x slab pairs x
    pstride x 32 bytes."""
    import oracle
    n, h, w, c, kh, kw, s, p = geom
    g = oracle.win_geometry(n, h, w, c, kh, kw, s, p, p)
    assert bs.tcw_act_bytes(n, h, w, c, kh, kw, s, p, bits) == (bits + 1) // 2 * g["nph"] * g["pairs"] * g["pstride"] * 32


@pytest.mark.parametrize("oc,kh,kw,c,w_bits", [(64, 3, 3, 64, 1), (100, 1, 1, 33, 2), (512, 3, 3, 512, 4), (4, 2, 3, 5, 3)])
def test_tcw_weight_size_matches_the_oracle_definition(lib, oc, kh, kw, c, w_bits):
    import numpy as np
    import oracle
    ref = oracle.conv2d_tcw_weights(np.zeros((oc, kh, kw, c), dtype=np.uint8), w_bits, 0)
    assert bs.conv2d_tcw_weight_bytes(oc, kh, kw, c, w_bits) == ref.size


def test_tcw_validation_before_launch(lib):
    # outside the window layout's domain: stride 3, unequal strides, a grid row wider than a tile
    assert bs.tcw_act_bytes(1, 12, 12, 8, 3, 3, 3, 1, 2) == 0
    assert bs.tcw_act_bytes(1, 8, 300, 8, 3, 3, 1, 1, 2) == 0
    conv = lib.bs_bitserial_conv2d_nhwc_tcw
    #                 act   A  enc  w     W  enc  out   n  h  w  c  oc kh kw sh sw ph pw stream
    assert conv(FAKE, 2, 0, FAKE, 1, 1, FAKE, 1, 8, 8, 8, 8, 3, 3, 1, 2, 1, 1, NULL) == 3
    assert b"stride" in lib.bs_last_error()
    assert conv(FAKE, 2, 0, FAKE, 1, 1, FAKE, 1, 8, 8, 8, 6, 3, 3, 1, 1, 1, 1, NULL) == 3   # oc % 4 != 0
    assert b"multiple of 4" in lib.bs_last_error()
    assert conv(FAKE, 4, 0, FAKE, 4, 0, FAKE, 1, 4, 4, 20000, 8, 3, 3, 1, 1, 1, 1, NULL) == 6  # FP4 bound
    assert conv(NULL, 2, 0, FAKE, 1, 1, FAKE, 1, 8, 8, 8, 8, 3, 3, 1, 1, 1, 1, NULL) == 1     # NULL operand
    # pack: output buffer too small, bad bit width
    pack = lib.bs_digitpack_win
    assert pack(FAKE, FAKE, 16, 1, 8, 8, 8, 3, 3, 1, 1, 1, 2, 0, NULL) == 8
    assert pack(FAKE, FAKE, 1 << 30, 1, 8, 8, 8, 3, 3, 1, 1, 1, 5, 0, NULL) == 2
