"""Pins of the CPU oracle to things other than itself (CPU only, -m "not gpu").

Every check here is independent of oracle/oracle.c's code:
  * Eq. 2 evaluated literally on bit-planes extracted here with
    Python integer bit operations and bin().count('1'), exhaustively on tiny vectors;
  * the north_star bipolar form popc(a&w) - popc(a&~w) per plane pair, exhaustively;
  * float64 torch.mm / torch.nn.functional.conv2d (exact: all partial sums are
    integers far below 2^53) on non-square, non-symmetric random inputs;
  * a second brute-force conv in Python with a different loop order;
  * closed forms (all-max interior/edge/corner, all-zero, code-0 bipolar);
  * invariants (stride-2 = subsampled stride-1, 1x1 conv = dense, plane
    decomposition, payload conservation and round trip of the packing);
  * hand-derived golden fixtures in tests/golden/ (each cites its passage).
A dropped term, a wrong sign, a wrong index/stride/pad, a transposed operand or a
kernel flip in the oracle fails at least one of them.
"""
import itertools
import json
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def popcount(x: int) -> int:
    return bin(x).count("1")


def planes(vec, bits):
    """Bit-plane i of a code vector as a Python int bit-vector (element t at bit t)."""
    out = []
    for i in range(bits):
        word = 0
        for t, v in enumerate(vec):
            if (int(v) >> i) & 1:
                word |= 1 << t
        out.append(word)
    return out


def eq2_unipolar(a, a_bits, w, w_bits):
    """PAPER.md:512 Eq. 2: sum_n sum_m popcount(x_n & y_m) * 2^(m+n)."""
    ap, wp = planes(a, a_bits), planes(w, w_bits)
    return sum(popcount(ap[i] & wp[j]) << (i + j) for i in range(a_bits) for j in range(w_bits))


def eq2_bipolar_literal(a, a_bits, w, w_bits):
    """north_star: per plane pair popc(a_i & w_j) - popc(a_i & ~w_j), weighted 2^(i+j)."""
    k = len(a)
    mask = (1 << k) - 1
    ap, wp = planes(a, a_bits), planes(w, w_bits)
    return sum((popcount(ap[i] & wp[j]) - popcount(ap[i] & (~wp[j] & mask))) << (i + j)
               for i in range(a_bits) for j in range(w_bits))


# --------------------------------------------------------------------------- golden
def test_golden_dot_examples():
    for c in _gold("dot_examples.json")["cases"]:
        got = oracle.dense(np.array([c["a"]]), c["a_bits"], np.array([c["w"]]), c["w_bits"], c["bipolar"])
        assert got.shape == (1, 1) and int(got[0, 0]) == c["out"], c["note"]


def test_golden_pack_examples():
    for c in _gold("pack_examples.json")["cases"]:
        got = oracle.bitpack(np.array(c["codes"]), c["bits"])
        assert got.dtype == np.uint32
        assert got.tolist() == c["packed"], c["note"]


def test_golden_conv_examples():
    for c in _gold("conv_examples.json")["cases"]:
        act = np.full((c["n"], c["h"], c["w"], c["c"]), c["act_fill"], np.uint8)
        wt = np.full((c["oc"], c["k"], c["k"], c["c"]), c["wt_fill"], np.uint8)
        out = oracle.conv2d_nhwc(act, c["a_bits"], wt, c["w_bits"], c["bipolar"],
                                 stride=(c["stride"],) * 2, pad=(c["pad"],) * 2)
        assert out.shape == (c["n"], c["oh"], c["ow"], c["oc"])
        if "out_fill" in c:
            assert (out == c["out_fill"]).all()
        else:
            oh, ow = c["oh"], c["ow"]
            assert (out[0, 1:oh - 1, 1:ow - 1] == c["interior"]).all()
            assert (out[0, 0, 1:ow - 1] == c["edge"]).all() and (out[0, 1:oh - 1, 0] == c["edge"]).all()
            for y, x in [(0, 0), (0, ow - 1), (oh - 1, 0), (oh - 1, ow - 1)]:
                assert (out[0, y, x] == c["corner"]).all()


def test_delta_kernel_reproduces_input():
    """a single 1 at the centre of a 3x3 kernel, pad 1, copies the input channel."""
    rng = np.random.default_rng(1)
    act = rng.integers(0, 4, (2, 5, 7, 3), dtype=np.uint8)
    for ch in range(3):
        wt = np.zeros((1, 3, 3, 3), np.uint8)
        wt[0, 1, 1, ch] = 1
        out = oracle.conv2d_nhwc(act, 2, wt, 1, False, stride=(1, 1), pad=(1, 1))
        np.testing.assert_array_equal(out[..., 0], act[..., ch].astype(np.int32))


def test_identity_matmul():
    """identity weights reproduce the activation rows."""
    rng = np.random.default_rng(2)
    a = rng.integers(0, 8, (5, 4), dtype=np.uint8)
    out = oracle.dense(a, 3, np.eye(4, dtype=np.uint8), 1, False)
    np.testing.assert_array_equal(out, a.astype(np.int32))


def test_table1_extents():
    from paper_1810_11066_b200.inputs import TABLE1
    g = _gold("table1_extents.json")["layers"]
    for name, row in g.items():
        L = TABLE1[int(name)]
        assert L.h == row["h"]
        assert oracle.conv_out_extent(L.h, L.k, L.s, L.pad) == row["oh"]
        assert row["oh"] ** 2 == row["M_b1"] and L.k * L.k * L.ic == row["K"]


# ----------------------------------------------------------------- Eq. 2 exhaustive
@pytest.mark.parametrize("a_bits,w_bits,k", [(2, 1, 3), (1, 2, 3), (2, 2, 2), (1, 1, 4), (3, 1, 2), (1, 3, 2)])
def test_eq2_exhaustive(a_bits, w_bits, k):
    """Oracle (plain integer definition) == Eq. 2 on bit-planes, for every code vector,
    unipolar, and == the literal bipolar plane-pair form, bipolar (readings R1-R3)."""
    avs = list(itertools.product(range(1 << a_bits), repeat=k))
    wvs = list(itertools.product(range(1 << w_bits), repeat=k))
    A = np.array(avs, np.uint8)
    W = np.array(wvs, np.uint8)
    uni = oracle.dense(A, a_bits, W, w_bits, False)
    bip = oracle.dense(A, a_bits, W, w_bits, True)
    for i, a in enumerate(avs):
        for j, w in enumerate(wvs):
            assert uni[i, j] == eq2_unipolar(a, a_bits, w, w_bits)
            assert bip[i, j] == eq2_bipolar_literal(a, a_bits, w, w_bits)


def test_weight_value_table():
    """Reading R2/R3: bipolar W1 codes {0,1} -> {-1,+1}; W2 {0,1,2,3} -> {-3,-1,+1,+3}."""
    assert [oracle.weight_value(c, 1, True) for c in range(2)] == [-1, 1]
    assert [oracle.weight_value(c, 2, True) for c in range(4)] == [-3, -1, 1, 3]
    assert [oracle.weight_value(c, 3, True) for c in range(8)] == [2 * c - 7 for c in range(8)]
    assert [oracle.weight_value(c, 2, False) for c in range(4)] == [0, 1, 2, 3]


# ------------------------------------------------------------- library routines
def _decode(w, w_bits, bipolar):
    w = w.astype(np.float64)
    return 2 * w - (2 ** w_bits - 1) if bipolar else w


@pytest.mark.parametrize("a_bits,w_bits,bipolar", [(1, 1, False), (2, 1, True), (2, 2, True), (4, 2, False), (8, 1, True), (3, 3, True)])
def test_dense_vs_torch_mm(a_bits, w_bits, bipolar):
    rng = np.random.default_rng(10 * a_bits + w_bits)
    m, n, k = 37, 29, 203
    a = rng.integers(0, 2 ** a_bits, (m, k), dtype=np.uint8)
    w = rng.integers(0, 2 ** w_bits, (n, k), dtype=np.uint8)
    got = oracle.dense(a, a_bits, w, w_bits, bipolar)
    ref = torch.from_numpy(a.astype(np.float64)) @ torch.from_numpy(_decode(w, w_bits, bipolar)).T
    np.testing.assert_array_equal(got, ref.numpy().astype(np.int64))


CONV_CASES = [
    # n, h, w, c, oc, kh, kw, sh, sw, ph, pw
    (2, 9, 7, 5, 3, 3, 3, 1, 1, 1, 1),
    (1, 8, 11, 33, 4, 3, 3, 2, 2, 1, 1),
    (3, 6, 5, 64, 2, 1, 1, 2, 2, 0, 0),
    (1, 7, 7, 3, 5, 3, 2, 1, 2, 0, 1),     # non-square kernel, mixed stride/pad
    (2, 5, 9, 17, 6, 2, 3, 3, 1, 2, 0),
]


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("a_bits,w_bits,bipolar", [(2, 1, True), (1, 2, False), (2, 2, True)])
def test_conv_vs_torch_conv2d(case, a_bits, w_bits, bipolar):
    n, h, w, c, oc, kh, kw, sh, sw, ph, pw = case
    rng = np.random.default_rng(sum(case) + a_bits)
    act = rng.integers(0, 2 ** a_bits, (n, h, w, c), dtype=np.uint8)
    wt = rng.integers(0, 2 ** w_bits, (oc, kh, kw, c), dtype=np.uint8)
    got = oracle.conv2d_nhwc(act, a_bits, wt, w_bits, bipolar, stride=(sh, sw), pad=(ph, pw))
    x = torch.from_numpy(act.astype(np.float64)).permute(0, 3, 1, 2)
    k_ = torch.from_numpy(_decode(wt, w_bits, bipolar)).permute(0, 3, 1, 2)
    ref = F.conv2d(x, k_, stride=(sh, sw), padding=(ph, pw)).permute(0, 2, 3, 1)
    np.testing.assert_array_equal(got, ref.numpy().astype(np.int64))


def _conv_bruteforce(act, wt, values, stride, pad):
    """Second independent loop order: taps outermost, scatter into outputs."""
    n, h, w, c = act.shape
    oc, kh, kw, _ = wt.shape
    sh, sw = stride
    ph, pw = pad
    oh, ow = (h + 2 * ph - kh) // sh + 1, (w + 2 * pw - kw) // sw + 1
    out = np.zeros((n, oh, ow, oc), np.int64)
    for ky in range(kh):
        for kx in range(kw):
            for ci in range(c):
                for o in range(oc):
                    v = int(values[o, ky, kx, ci])
                    for b in range(n):
                        for oy in range(oh):
                            iy = oy * sh + ky - ph
                            if not 0 <= iy < h:
                                continue
                            for ox in range(ow):
                                ix = ox * sw + kx - pw
                                if 0 <= ix < w:
                                    out[b, oy, ox, o] += int(act[b, iy, ix, ci]) * v
    return out


def test_conv_vs_bruteforce_second_loop_order():
    rng = np.random.default_rng(7)
    act = rng.integers(0, 4, (1, 5, 6, 3), dtype=np.uint8)
    wt = rng.integers(0, 4, (2, 3, 3, 3), dtype=np.uint8)
    for bip in (False, True):
        vals = np.vectorize(lambda c: oracle.weight_value(int(c), 2, bip))(wt)
        got = oracle.conv2d_nhwc(act, 2, wt, 2, bip, stride=(2, 1), pad=(1, 1))
        np.testing.assert_array_equal(got, _conv_bruteforce(act, wt, vals, (2, 1), (1, 1)))


# ------------------------------------------------------------------- invariants
def test_stride2_is_subsampled_stride1():
    rng = np.random.default_rng(3)
    act = rng.integers(0, 4, (2, 9, 9, 10), dtype=np.uint8)
    wt = rng.integers(0, 2, (4, 3, 3, 10), dtype=np.uint8)
    s1 = oracle.conv2d_nhwc(act, 2, wt, 1, True, stride=(1, 1), pad=(1, 1))
    s2 = oracle.conv2d_nhwc(act, 2, wt, 1, True, stride=(2, 2), pad=(1, 1))
    np.testing.assert_array_equal(s2, s1[:, ::2, ::2])


def test_1x1_conv_is_dense():
    """1x1 stride-1 pad-0 conv equals dense on reshaped operands."""
    rng = np.random.default_rng(4)
    act = rng.integers(0, 4, (2, 4, 5, 40), dtype=np.uint8)
    wt = rng.integers(0, 4, (7, 1, 1, 40), dtype=np.uint8)
    conv = oracle.conv2d_nhwc(act, 2, wt, 2, True)
    dense = oracle.dense(act.reshape(-1, 40), 2, wt.reshape(7, 40), 2, True)
    np.testing.assert_array_equal(conv.reshape(-1, 7), dense)


def test_plane_decomposition_and_bipolar_identity():
    """out(a) = sum_i 2^i out(a_i) (Eq. 2 linearity in the activation planes) and
    bipolar = 2*unipolar - (2^W - 1) * sum(a)."""
    rng = np.random.default_rng(5)
    a = rng.integers(0, 16, (6, 77), dtype=np.uint8)
    w = rng.integers(0, 4, (5, 77), dtype=np.uint8)
    full = oracle.dense(a, 4, w, 2, False)
    parts = sum((oracle.dense((a >> i) & 1, 1, w, 2, False).astype(np.int64) << i) for i in range(4))
    np.testing.assert_array_equal(full, parts)
    bip = oracle.dense(a, 4, w, 2, True).astype(np.int64)
    np.testing.assert_array_equal(bip, 2 * full - 3 * a.astype(np.int64).sum(1, keepdims=True))


def test_closed_forms():
    z = oracle.dense(np.zeros((3, 50), np.uint8), 2, np.ones((4, 50), np.uint8), 1, True)
    assert (z == 0).all()
    a = np.full((2, 50), 3, np.uint8)
    neg = oracle.dense(a, 2, np.zeros((3, 50), np.uint8), 2, True)
    assert (neg == -3 * 150).all()
    mx = oracle.dense(np.full((1, 1000), 15, np.uint8), 4, np.full((1, 1000), 3, np.uint8), 2, False)
    assert mx[0, 0] == 1000 * 15 * 3


# ---------------------------------------------------------------------- packing
def _unpack(p, k):
    bits, rows, kw = p.shape
    out = np.zeros((rows, k), np.int64)
    for b in range(bits):
        for r in range(rows):
            for j in range(k):
                out[r, j] |= ((int(p[b, r, j // 32]) >> (j % 32)) & 1) << b
    return out


@pytest.mark.parametrize("rows,k,bits", [(3, 1, 1), (2, 31, 2), (4, 32, 3), (2, 33, 2), (3, 100, 4), (1, 64, 8), (2, 130, 1)])
def test_pack_roundtrip_conservation_pad(rows, k, bits):
    rng = np.random.default_rng(rows * 1000 + k + bits)
    x = rng.integers(0, 2 ** bits, (rows, k), dtype=np.uint8)
    p = oracle.bitpack(x, bits)
    kw = (k + 31) // 32
    assert p.shape == (bits, rows, kw + (kw & 1))
    np.testing.assert_array_equal(_unpack(p, k), x)
    # payload conservation: total set bits = sum of popcounts of codes
    assert sum(popcount(int(v)) for v in p.ravel()) == sum(popcount(int(v)) for v in x.ravel())
    # pad bits / pad words are zero
    for b in range(bits):
        for r in range(rows):
            for j in range(p.shape[2]):
                lo = 32 * j
                valid = max(0, min(32, k - lo))
                assert int(p[b, r, j]) >> valid == 0


def test_pack_eq2_from_packed_words():
    """Eq. 2 evaluated on the oracle's packed words equals the oracle's dense product:
    ties the packed layout to the arithmetic the GPU path performs."""
    rng = np.random.default_rng(9)
    a = rng.integers(0, 4, (3, 70), dtype=np.uint8)
    w = rng.integers(0, 2, (4, 70), dtype=np.uint8)
    pa, pw = oracle.bitpack(a, 2), oracle.bitpack(w, 1)
    ref = oracle.dense(a, 2, w, 1, False)
    for m in range(3):
        for n in range(4):
            s = sum(popcount(int(pa[i, m, j]) & int(pw[0, n, j])) << i
                    for i in range(2) for j in range(pa.shape[2]))
            assert s == ref[m, n]


def test_rejections():
    with pytest.raises(ValueError):
        oracle.dense(np.full((1, 4), 4, np.uint8), 2, np.zeros((1, 4), np.uint8), 1, False)  # code out of range
    with pytest.raises(ValueError):
        oracle.conv2d_nhwc(np.zeros((1, 2, 2, 1), np.uint8), 1, np.zeros((1, 3, 3, 1), np.uint8), 1, False)  # empty
    with pytest.raises(ValueError):  # accumulator bound K*(2^8-1)^2 >= 2^31
        oracle.dense(np.zeros((1, 40000), np.uint8), 8, np.zeros((1, 40000), np.uint8), 8, False)


# ----------------------------------------------------- encodings
def eq2_signed_literal(a, a_bits, a_signed, w, w_bits, w_signed):
    """PAPER.md:517 "Equation 2 can be modified to support signed data by weighting
    binary dotproducts by their sign": two's complement, the top plane of a signed
    operand carries sign -1, every plane pair popc(x_n & y_m) * s_n * s_m * 2^(n+m)."""
    ap, wp = planes(a, a_bits), planes(w, w_bits)
    sa = [(-1 if (a_signed and i == a_bits - 1) else 1) for i in range(a_bits)]
    sw = [(-1 if (w_signed and j == w_bits - 1) else 1) for j in range(w_bits)]
    return sum(sa[i] * sw[j] * (popcount(ap[i] & wp[j]) << (i + j)) for i in range(a_bits) for j in range(w_bits))


def eq2_xnor_literal(a, a_bits, w, w_bits):
    """bipolar (-1/+1) data, "bitwise xnor replaces bitwise and": for
    +/-1 digit vectors x_n, y_m of length K, x_n . y_m = 2 popc(~(x_n ^ y_m)) - K, and
    the multi-bit value is sum_n sum_m 2^(n+m) x_n . y_m (Eq. 2 with that dot)."""
    k = len(a)
    mask = (1 << k) - 1
    ap, wp = planes(a, a_bits), planes(w, w_bits)
    return sum((2 * popcount(~(ap[i] ^ wp[j]) & mask) - k) << (i + j) for i in range(a_bits) for j in range(w_bits))


def test_code_value_tables():
    """Encodings: signed = two's complement; bipolar = 2 code - (2^bits - 1); unsigned."""
    assert [oracle.code_value(c, 2, oracle.SIGNED) for c in range(4)] == [0, 1, -2, -1]
    assert [oracle.code_value(c, 3, oracle.SIGNED) for c in range(8)] == [0, 1, 2, 3, -4, -3, -2, -1]
    assert [oracle.code_value(c, 1, oracle.SIGNED) for c in range(2)] == [0, -1]
    assert [oracle.code_value(c, 4, oracle.BIPOLAR) for c in range(16)] == [2 * c - 15 for c in range(16)]
    assert [oracle.code_value(c, 3, oracle.UNSIGNED) for c in range(8)] == list(range(8))


@pytest.mark.parametrize("a_bits,w_bits,k", [(2, 1, 3), (1, 2, 3), (2, 2, 2), (3, 1, 2), (1, 1, 4)])
def test_encodings_exhaustive(a_bits, w_bits, k):
    """Every code vector pair: the encoded oracle equals (1) the sign-weighted Eq. 2 for
    each signed/unsigned combination, (2) the XNOR form for both operands bipolar,
    (3) the literal bipolar-weight form and the plain oracle for unsigned activations."""
    avs = list(itertools.product(range(1 << a_bits), repeat=k))
    wvs = list(itertools.product(range(1 << w_bits), repeat=k))
    A = np.array(avs, np.uint8)
    W = np.array(wvs, np.uint8)
    U, B, S = oracle.UNSIGNED, oracle.BIPOLAR, oracle.SIGNED
    res = {(ae, we): oracle.dense_enc(A, a_bits, ae, W, w_bits, we) for ae in (U, B, S) for we in (U, B, S)}
    np.testing.assert_array_equal(res[(U, U)], oracle.dense(A, a_bits, W, w_bits, False))
    np.testing.assert_array_equal(res[(U, B)], oracle.dense(A, a_bits, W, w_bits, True))
    for i, a in enumerate(avs):
        for j, w in enumerate(wvs):
            assert res[(S, S)][i, j] == eq2_signed_literal(a, a_bits, True, w, w_bits, True)
            assert res[(S, U)][i, j] == eq2_signed_literal(a, a_bits, True, w, w_bits, False)
            assert res[(U, S)][i, j] == eq2_signed_literal(a, a_bits, False, w, w_bits, True)
            assert res[(B, B)][i, j] == eq2_xnor_literal(a, a_bits, w, w_bits)


def _decode_enc(x, bits, enc):
    x = x.astype(np.float64)
    if enc == oracle.BIPOLAR:
        return 2 * x - (2 ** bits - 1)
    if enc == oracle.SIGNED:
        return np.where(x >= 2 ** (bits - 1), x - 2 ** bits, x)
    return x


@pytest.mark.parametrize("a_enc,w_enc", [(1, 1), (2, 2), (2, 0), (0, 2), (1, 2), (2, 1), (1, 0)])
def test_encoded_dense_and_conv_vs_torch(a_enc, w_enc):
    """Library pin: float64 torch mm / conv2d (zero padding = value 0) on decoded values."""
    rng = np.random.default_rng(7 * a_enc + w_enc)
    for a_bits, w_bits in ((2, 1), (3, 2), (1, 1), (4, 3)):
        a = rng.integers(0, 2 ** a_bits, (23, 131), dtype=np.uint8)
        w = rng.integers(0, 2 ** w_bits, (17, 131), dtype=np.uint8)
        got = oracle.dense_enc(a, a_bits, a_enc, w, w_bits, w_enc)
        ref = torch.from_numpy(_decode_enc(a, a_bits, a_enc)) @ torch.from_numpy(_decode_enc(w, w_bits, w_enc)).T
        np.testing.assert_array_equal(got, ref.numpy().astype(np.int64))
        for case in CONV_CASES[:3]:
            n, h, w_, c, oc, kh, kw, sh, sw, ph, pw = case
            act = rng.integers(0, 2 ** a_bits, (n, h, w_, c), dtype=np.uint8)
            wt = rng.integers(0, 2 ** w_bits, (oc, kh, kw, c), dtype=np.uint8)
            got = oracle.conv2d_nhwc_enc(act, a_bits, a_enc, wt, w_bits, w_enc, stride=(sh, sw), pad=(ph, pw))
            x = torch.from_numpy(_decode_enc(act, a_bits, a_enc)).permute(0, 3, 1, 2)
            k_ = torch.from_numpy(_decode_enc(wt, w_bits, w_enc)).permute(0, 3, 1, 2)
            ref = F.conv2d(x, k_, stride=(sh, sw), padding=(ph, pw)).permute(0, 2, 3, 1)
            np.testing.assert_array_equal(got, ref.numpy().astype(np.int64))


def test_encoded_closed_forms():
    """Both bipolar, all codes max (every digit +1): each output = K (2^A-1)(2^W-1);
    signed all-ones codes are -1: each output = K; signed min code x max."""
    k = 77
    a = np.full((3, k), 3, np.uint8)
    w = np.full((2, k), 1, np.uint8)
    assert (oracle.dense_enc(a, 2, 1, w, 1, 1) == k * 3 * 1).all()
    assert (oracle.dense_enc(a, 2, 2, np.full((2, k), 3, np.uint8), 2, 2) == k).all()  # (-1)(-1)
    assert (oracle.dense_enc(np.full((1, k), 2, np.uint8), 2, 2, np.full((1, k), 1, np.uint8), 2, 2) == -2 * k).all()
    with pytest.raises(ValueError):
        oracle.dense_enc(a, 2, 3, w, 1, 0)


# ------------------------------------------------------------- digit packing (R21/R24)
def test_e2m1_decode_table():
    """The 4-bit E2M1 format's magnitudes are {0, 0.5, 1, 1.5, 2, 3, 4, 6} (codes 0-7), the
    sign bit negates (codes 8-15): the format definition the digit fields are written in."""
    twice = [oracle.e2m1_twice(x) for x in range(16)]
    assert twice[:8] == [0, 1, 2, 3, 4, 6, 8, 12]
    assert twice[8:] == [-v for v in twice[:8]]


def test_digitpack_golden():
    with open(os.path.join(GOLD, "digit_examples.json")) as f:
        gold = json.load(f)
    for case in gold["cases"]:
        x = np.array(case["codes"], dtype=np.uint8)
        got = oracle.digitpack(x, case["bits"], case["enc"])
        assert got.shape == (len(case["digits"]), x.shape[0], case["row_bytes"])
        for d, want in enumerate(case["digits"]):
            np.testing.assert_array_equal(got[d, 0, :len(want)], want, err_msg=case["note"])
            assert not got[d, 0, len(want):].any(), case["note"]


@pytest.mark.parametrize("bits", [1, 2, 3, 4])
@pytest.mark.parametrize("enc", [0, 1, 2])
def test_digitpack_digits_sum_to_code_value(bits, enc):
    """Exhaustively over every code: sum_d 4^d * value(field_d) is the code's value in its
    encoding (Eq. 2's plane weights 2^i regrouped as 4^d (2^0, 2^1) per digit) — read back
    from the packed bytes with Python bit operations, independent of the C digit rules."""
    codes = np.arange(1 << bits, dtype=np.uint8).reshape(1, -1)
    got = oracle.digitpack(codes, bits, enc)
    for t, code in enumerate(codes[0]):
        total = 0
        for d in range(got.shape[0]):
            nib = (int(got[d, 0, t // 2]) >> (4 * (t % 2))) & 0xF
            total += 4 ** d * oracle.e2m1_twice(nib)
        if enc == 1:
            want = sum((1 << j) * (2 * ((int(code) >> j) & 1) - 1) for j in range(bits))
        elif enc == 2:
            want = int(code) - (1 << bits) if code >= 1 << (bits - 1) else int(code)
        else:
            want = int(code)
        assert total == want, (bits, enc, int(code))


def test_digitpack_unsigned_fields_are_bit_planes():
    """Unsigned digit fields hold exactly the two bit planes of the packed layout: field bit
    0 = plane 2d, bit 1 = plane 2d+1 (the same element order as oracle.bitpack), bits 2-3
    zero; the zero tail past k matches the packed rows' zero pad bits."""
    g = np.random.default_rng(7)
    for bits, rows, k in ((2, 5, 70), (4, 3, 33), (3, 4, 128), (1, 2, 5)):
        x = g.integers(0, 1 << bits, size=(rows, k), dtype=np.uint8)
        dig = oracle.digitpack(x, bits, 0)
        planes = oracle.bitpack(x, bits)
        kwp = planes.shape[2]
        assert dig.shape[2] == 16 * kwp
        for d in range(dig.shape[0]):
            for r in range(rows):
                for t in range(32 * kwp):
                    nib = (int(dig[d, r, t // 2]) >> (4 * (t % 2))) & 0xF
                    lo = (int(planes[2 * d, r, t // 32]) >> (t % 32)) & 1
                    hi = (int(planes[2 * d + 1, r, t // 32]) >> (t % 32)) & 1 if 2 * d + 1 < bits else 0
                    assert nib == lo | (hi << 1), (bits, d, r, t)


def test_digitpack_dot_product_matches_dense_enc():
    """Eq. 2 from the digit fields: sum_{d,e} 4^(d+e) sum_k v_a[k,d] v_w[k,e] equals the
    oracle's plain dense product, for every encoding pair (a dropped digit, a wrong digit
    weight or a wrong sign rule fails here)."""
    g = np.random.default_rng(11)
    for a_bits, w_bits in ((2, 1), (3, 2), (4, 4), (1, 3)):
        for a_enc in (0, 1, 2):
            for w_enc in (0, 1, 2):
                a = g.integers(0, 1 << a_bits, size=(3, 45), dtype=np.uint8)
                w = g.integers(0, 1 << w_bits, size=(4, 45), dtype=np.uint8)
                da, dw = oracle.digitpack(a, a_bits, a_enc), oracle.digitpack(w, w_bits, w_enc)

                def vals(p):  # [D][rows][elements] digit values decoded from the fields
                    lo = np.vectorize(oracle.e2m1_twice)(p & 0xF)
                    hi = np.vectorize(oracle.e2m1_twice)(p >> 4)
                    return np.stack([lo, hi], axis=-1).reshape(p.shape[0], p.shape[1], -1).astype(np.int64)
                va, vw = vals(da), vals(dw)
                out = np.zeros((3, 4), dtype=np.int64)
                for d in range(va.shape[0]):
                    for e in range(vw.shape[0]):
                        out += 4 ** (d + e) * (va[d] @ vw[e].T)
                np.testing.assert_array_equal(out, oracle.dense_enc(a, a_bits, a_enc, w, w_bits, w_enc))


# ---------------------------------------------------------------- window layout (R26)
def test_win_layout_golden():
    """Hand-derived window-layout bytes (tests/golden/win_examples.json, each case cites R26)."""
    for case in _gold("win_examples.json")["cases"]:
        x = np.array(case["codes"], dtype=np.uint8)
        got = oracle.digitpack_win(x, case["bits"], case["enc"], case["kh"], case["kw"], case["stride"],
                                   case["pad"], case["pad"])
        d, f, cs, nq, nb = case["shape"]
        assert got.shape[:3] == (d, f, cs), case["note"]
        want = np.zeros_like(got)
        for dd, ff, cc, q, b, v in case["nonzero"]:
            want[dd, ff, cc, q, b] = v
        np.testing.assert_array_equal(got, want, err_msg=case["note"])


def _e2m1_vals(p):
    """Digit values of a byte array's two nibbles, last axis doubled: element 2b = low nibble."""
    lo = np.vectorize(oracle.e2m1_twice)(p & 0xF)
    hi = np.vectorize(oracle.e2m1_twice)(p >> 4)
    return np.stack([lo, hi], axis=-1).reshape(*p.shape[:-1], -1).astype(np.int64)


WIN_CASES = [  # (n, h, w, c, oc, kh, kw, stride, pad, a_bits, w_bits)
    (2, 5, 4, 40, 24, 3, 3, 1, 1, 2, 1),
    (1, 6, 7, 33, 70, 3, 3, 2, 1, 3, 2),
    (2, 6, 6, 64, 8, 1, 1, 2, 0, 2, 2),
    (1, 5, 6, 20, 5, 2, 3, 1, 0, 4, 1),
    (1, 7, 5, 96, 130, 3, 2, 2, 2, 1, 3),
    (3, 3, 3, 16, 4, 3, 3, 1, 2, 2, 1),
]


@pytest.mark.parametrize("case", WIN_CASES)
@pytest.mark.parametrize("enc", [(0, 0), (0, 1), (1, 1), (2, 2)])
def test_win_layout_conv_brute_force(case, enc):
    """Convolution evaluated FROM the two window layouts with the tap-offset rule of R26 —
    out[q] = sum_{d,e} 4^(d+e) sum_tap sum_ch A_d[phase(tap)][q + off(tap)][ch] W_e[o][tap][ch],
    q = (img*hg + oy)*wg + ox, off = (ky//s)*wg + kx//s, each 32-byte row read back through the
    half exchange of rows with bit 2 set — decoded here with Python E2M1 arithmetic, equals the
    oracle's plain NHWC convolution (a wrong phase, offset, padding position, slab order,
    swizzle or filter block fails it)."""
    n, h, w, c, oc, kh, kw, s, pad, a_bits, w_bits = case
    a_enc, w_enc = enc
    g = np.random.default_rng(hash(case) % 1000 + 17 * a_enc + w_enc)
    act = g.integers(0, 1 << a_bits, size=(n, h, w, c), dtype=np.uint8)
    wt = g.integers(0, 1 << w_bits, size=(oc, kh, kw, c), dtype=np.uint8)
    geo = oracle.win_geometry(n, h, w, c, kh, kw, s, pad, pad)

    def unswizzle(b):   # [..., rows, 32]: exchange the halves back where bit 2 of the row is set
        r = np.arange(b.shape[-2])
        sw = ((r >> 2) & 1).astype(bool)
        out = b.copy()
        out[..., sw, :16], out[..., sw, 16:] = b[..., sw, 16:], b[..., sw, :16]
        return out
    A = _e2m1_vals(unswizzle(oracle.digitpack_win(act, a_bits, a_enc, kh, kw, s, pad, pad)))  # [D][f][p][q][64]
    Wt = _e2m1_vals(unswizzle(oracle.conv2d_tcw_weights(wt, w_bits, w_enc)))                  # [nb][p][e][tap][r][64]
    nblk, pairs, De, taps, bn, _ = Wt.shape
    Wl = Wt.transpose(2, 0, 4, 3, 1, 5).reshape(De, nblk * bn, taps, pairs * 64)             # [e][o][tap][ch]
    A = A.transpose(0, 1, 3, 2, 4).reshape(A.shape[0], A.shape[1], A.shape[3], -1)            # [D][f][q][ch]
    hg, wg, oh, ow = geo["hg"], geo["wg"], geo["oh"], geo["ow"]
    q = ((np.arange(n)[:, None, None] * hg + np.arange(oh)[None, :, None]) * wg + np.arange(ow)[None, None, :]).ravel()
    out = np.zeros((q.size, nblk * bn), dtype=np.int64)
    for d in range(A.shape[0]):
        for e in range(De):
            for ky in range(kh):
                for kx in range(kw):
                    f = geo["phases"].index((ky % s) * s + kx % s)
                    off = (ky // s) * wg + kx // s
                    out += 4 ** (d + e) * (A[d, f, q + off] @ Wl[e, :, ky * kw + kx].T)
    want = oracle.conv2d_nhwc_enc(act, a_bits, a_enc, wt, w_bits, w_enc, stride=(s, s), pad=(pad, pad))
    np.testing.assert_array_equal(out[:, :oc].reshape(want.shape), want)
    assert not out[:, oc:].any()  # filters past oc (block padding) are zero


def test_win_layout_zero_outside_image():
    """Every window-layout entry that is padding, junk grid position or tail is zero, and the
    number of non-zero slab entries equals the number of (pixel, slab) pairs the phases keep
    (stride 1: every pixel once)."""
    g = np.random.default_rng(3)
    act = g.integers(1, 4, size=(2, 5, 6, 32), dtype=np.uint8)   # codes >= 1: every real pixel non-zero
    lay = oracle.digitpack_win(act, 2, 0, 3, 3, 1, 1, 1)      # [1][1][1][pstride][32]
    geo = oracle.win_geometry(2, 5, 6, 32, 3, 3, 1, 1, 1)
    nz = lay[0, 0, 0].any(axis=1)
    assert nz.sum() == 2 * 5 * 6
    q = np.nonzero(nz)[0]
    assert q.max() < geo["gpix"]
    rem = q % (geo["hg"] * geo["wg"])
    gy, gx = rem // geo["wg"], rem % geo["wg"]
    assert gy.min() == 1 and gy.max() == 5 and gx.min() == 1 and gx.max() == 6
    # c = 32: the pair's second (pad) slab is zero: per row exactly one 16-byte half is non-zero,
    # the first half unless bit 2 of q is set
    half1 = lay[0, 0, 0, q, 16:].any(axis=1)
    np.testing.assert_array_equal(half1, ((q >> 2) & 1).astype(bool))
    assert not (lay[0, 0, 0, q, :16].any(axis=1) & half1).any()
