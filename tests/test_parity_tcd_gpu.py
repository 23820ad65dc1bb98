"""GPU parity of the digit-packed path (digit.cu + the TMA-fed tensor-core kernel tcd_conv.cu)
against the CPU oracle, element by element, zero tolerance (R14).  Expected values
only come from oracle/; inputs from paper_1810_11066_b200.inputs."""
import numpy as np
import pytest
import torch

import oracle
import paper_1810_11066_b200 as bs
from paper_1810_11066_b200 import inputs

pytestmark = pytest.mark.gpu
DEV = "cuda"


def wdig_conv(wt, w_bits, w_enc):
    """Weight digits of OHWI codes through the library (bitpack + prepare)."""
    oc, kh, kw, c = wt.shape
    wp = bs.bitpack(wt.reshape(oc * kh * kw, c).to(DEV), w_bits)
    return bs.conv2d_tcd_prepare_weights(wp, w_bits, w_enc, oc, kh, kw, c)


def run_conv(act, a_bits, a_enc, wt, w_bits, w_enc, stride, pad):
    n, h, w, c = act.shape
    oc, kh, kw, _ = wt.shape
    ad = bs.digitpack(act.reshape(-1, c).to(DEV), a_bits, a_enc)
    wd = wdig_conv(wt, w_bits, w_enc)
    return bs.bitserial_conv2d_nhwc_tcd(ad, a_bits, wd, w_bits, n, h, w, c, oc, kh, kw, stride, pad, a_enc=a_enc,
                                        w_enc=w_enc)


# ------------------------------------------------------------------ digit packing
@pytest.mark.parametrize("rows,k,bits,enc", [(1, 1, 1, 0), (3, 31, 2, 1), (5, 32, 2, 0), (7, 33, 3, 2), (4, 100, 4, 1),
                                             (3136, 64, 2, 1), (513, 4096, 2, 0), (1000, 48, 4, 2), (37, 3, 2, 1),
                                             (11, 576, 3, 0), (6, 96, 1, 1), (9, 160, 4, 0)])
def test_digitpack_parity(rows, k, bits, enc):
    g = inputs.gen(rows * 7919 + k * 31 + bits + 5 * enc)
    x = inputs.codes((rows, k), bits, g)
    got = bs.digitpack(x.to(DEV), bits, enc).cpu().numpy()
    np.testing.assert_array_equal(got, oracle.digitpack(x.numpy(), bits, enc))


def test_digitpack_group_parity():
    g = inputs.gen(77)
    xs = [inputs.codes(s, 2, g) for s in ((3136 * 3, 64), (784 * 2, 128), (49, 512), (17, 33), (5, 3))]
    outs = bs.digitpack_group([x.to(DEV) for x in xs], 2, bs.A_BIPOLAR)
    for x, o in zip(xs, outs):
        np.testing.assert_array_equal(o.cpu().numpy(), oracle.digitpack(x.numpy(), 2, bs.A_BIPOLAR))


@pytest.mark.parametrize("w_bits,w_enc", [(1, 0), (1, 1), (2, 1), (3, 2), (4, 0)])
def test_weight_digits_match_digitpack(w_bits, w_enc):
    """Prepared weight digits = the digit packing of every (filter, tap) channel row."""
    for oc, kh, kw, c in ((5, 3, 3, 33), (64, 3, 3, 64), (7, 1, 1, 100), (3, 2, 3, 192)):
        g = inputs.gen(oc * 13 + c + w_bits)
        wt = inputs.codes((oc, kh, kw, c), w_bits, g)
        ref = oracle.digitpack(wt.reshape(oc * kh * kw, c).numpy(), w_bits, w_enc)  # [P][oc*taps][rb]
        row = kh * kw * ref.shape[2]
        rpad = (row + 127) // 128 * 128  # rows zero-padded to 128-byte multiples
        got = wdig_conv(wt, w_bits, w_enc).cpu().numpy().reshape(ref.shape[0], oc, rpad)
        np.testing.assert_array_equal(got[:, :, :row], ref.reshape(ref.shape[0], oc, row))
        assert not got[:, :, row:].any()


# ------------------------------------------------------------------ conv
# (n, h, w, c, oc, kh, kw, stride, pad): several tiles + ragged tails; every channel-block width
# (C = 3/33/64 -> 32-byte pieces, 96/128 -> 64, 192 -> 3 x 32, 256/512 -> 128, 320 -> 5 x 32);
# strides 1-3, pads 0-2, non-square kernels, a kernel larger than the image, OC % 4 != 0
CONV_CASES = [
    (2, 9, 11, 33, 20, 3, 3, 1, 1),
    (1, 12, 10, 96, 100, 3, 3, 2, 1),
    (3, 7, 7, 64, 64, 1, 1, 1, 0),
    (2, 14, 14, 128, 130, 3, 3, 1, 1),
    (1, 15, 13, 192, 64, 3, 3, 2, 1),
    (2, 8, 8, 256, 256, 3, 3, 1, 1),
    (1, 9, 9, 320, 72, 3, 3, 3, 2),
    (2, 7, 7, 512, 96, 3, 3, 1, 1),
    (4, 11, 11, 3, 17, 5, 3, 1, 2),
    (1, 5, 6, 64, 36, 7, 7, 1, 3),
    (2, 56, 56, 64, 128, 1, 1, 2, 0),
    (1, 28, 28, 128, 256, 3, 3, 2, 1),
    (3, 5, 5, 40, 10, 2, 2, 2, 0),
]


@pytest.mark.parametrize("case", CONV_CASES, ids=lambda c: "x".join(map(str, c)))
@pytest.mark.parametrize("a_bits,w_bits", [(2, 1), (1, 1), (2, 2), (4, 2), (3, 4)])
def test_conv_tcd_parity(case, a_bits, w_bits):
    n, h, w, c, oc, kh, kw, s, p = case
    for w_enc in (bs.UNIPOLAR, bs.BIPOLAR):
        g = inputs.gen(n * 1000 + h * 37 + c * 7 + oc + 11 * a_bits + w_bits + w_enc)
        act = inputs.codes((n, h, w, c), a_bits, g)
        wt = inputs.codes((oc, kh, kw, c), w_bits, g)
        ref = oracle.conv2d_nhwc_enc(act.numpy(), a_bits, 0, wt.numpy(), w_bits, w_enc, stride=(s, s), pad=(p, p))
        got = run_conv(act, a_bits, 0, wt, w_bits, w_enc, s, p)
        np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"{case} A{a_bits}W{w_bits} w_enc={w_enc}")


ENC_PAIRS = [(a, w) for a in (bs.A_UNSIGNED, bs.A_BIPOLAR, bs.A_SIGNED) for w in (bs.UNIPOLAR, bs.BIPOLAR, bs.SIGNED)]


@pytest.mark.parametrize("a_enc,w_enc", ENC_PAIRS)
@pytest.mark.parametrize("a_bits,w_bits", [(1, 1), (2, 1), (2, 2), (3, 2), (4, 3), (1, 4)])
def test_conv_tcd_encodings(a_enc, w_enc, a_bits, w_bits):
    """Every (activation, weight) encoding — both bipolar is the XNOR form,
    signed the sign-weighted Eq. 2 — with padding (value 0 in every
    encoding), stride 2, channel tails and ragged M / OC."""
    for (n, h, w, c, oc, kh, kw, s, p) in ((2, 9, 11, 33, 20, 3, 3, 1, 1), (1, 12, 10, 96, 100, 3, 3, 2, 1)):
        g = inputs.gen(n * 1000 + c + 7 * a_enc + 3 * w_enc + 11 * a_bits + w_bits)
        act = inputs.codes((n, h, w, c), a_bits, g)
        wt = inputs.codes((oc, kh, kw, c), w_bits, g)
        ref = oracle.conv2d_nhwc_enc(act.numpy(), a_bits, a_enc, wt.numpy(), w_bits, w_enc, stride=(s, s), pad=(p, p))
        got = run_conv(act, a_bits, a_enc, wt, w_bits, w_enc, s, p)
        np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"c={c} a_enc={a_enc} w_enc={w_enc}")


def test_conv_tcd_group_matches_oracle():
    """The ResNet-18 body layers (Table 1) at batch 2 in ONE grouped launch."""
    layers = [inputs.TABLE1[i] for i in inputs.BASELINE_LAYERS]
    convs, refs = [], []
    for L in layers:
        act, wt = inputs.conv_operands(L, 2, 2, 1, seed=inputs.seed_for(3, 2, 1, "bipolar", L.name))
        refs.append(oracle.conv2d_nhwc_enc(act.numpy(), 2, 0, wt.numpy(), 1, 1, stride=(L.s, L.s),
                                           pad=(L.pad, L.pad)))
        convs.append(dict(act_dig=bs.digitpack(act.reshape(-1, L.ic).to(DEV), 2), w_dig=wdig_conv(wt, 1, 1), n=2,
                          h=L.h, w=L.w, c=L.ic, oc=L.oc, kh=L.k, kw=L.k, stride=L.s, pad=L.pad, w_enc=1))
    for idx in (range(5), range(5, len(convs)), range(len(convs))):
        outs = bs.bitserial_conv2d_nhwc_tcd_group([convs[i] for i in idx], 2, 1)
        for i, o in zip(idx, outs):
            np.testing.assert_array_equal(o.cpu().numpy(), refs[i], err_msg=f"layer {layers[i].name}")


def test_conv_tcd_sentinel_bands():
    """Outputs written between guard bands: nothing outside [out, out + M*oc) is touched."""
    n, h, w, c, oc, kh, kw, s, p = (3, 9, 7, 64, 36, 3, 3, 1, 1)
    g = inputs.gen(4242)
    act = inputs.codes((n, h, w, c), 2, g)
    wt = inputs.codes((oc, kh, kw, c), 1, g)
    ref = oracle.conv2d_nhwc_enc(act.numpy(), 2, 0, wt.numpy(), 1, 1, stride=(s, s), pad=(p, p))
    for oc_ in (36, 34):  # TMA-store and scalar epilogues
        wt_ = wt[:oc_].contiguous()
        ref_ = ref[..., :oc_]
        numel = ref_.size
        buf = torch.full((numel + 2 * 4096,), 0x5A5A5A5A, dtype=torch.int32, device=DEV)
        out = buf[4096:4096 + numel].view(ref_.shape)
        ad = bs.digitpack(act.reshape(-1, c).to(DEV), 2)
        bs.bitserial_conv2d_nhwc_tcd(ad, 2, wdig_conv(wt_, 1, 1), 1, n, h, w, c, oc_, kh, kw, s, p, out=out, w_enc=1)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(out.cpu().numpy(), ref_)
        assert bool((buf[:4096] == 0x5A5A5A5A).all()) and bool((buf[4096 + numel:] == 0x5A5A5A5A).all())


def test_conv_tcd_resnet_b256_sampled():
    """BASELINE configs[3] at full size (batch 256, A2W1 bipolar) through the grouped launch
    the bench times; images {0, 97, 255} of every layer against the oracle."""
    layers = [inputs.TABLE1[i] for i in inputs.BASELINE_LAYERS]
    convs, samples = [], []
    for L in layers:
        act, wt = inputs.conv_operands(L, 256, 2, 1, seed=inputs.seed_for(3, 2, 1, "bipolar", L.name))
        convs.append(dict(act_dig=bs.digitpack(act.reshape(-1, L.ic).to(DEV), 2), w_dig=wdig_conv(wt, 1, 1), n=256,
                          h=L.h, w=L.w, c=L.ic, oc=L.oc, kh=L.k, kw=L.k, stride=L.s, pad=L.pad, w_enc=1))
        samples.append((act, wt, L))
    outs = bs.bitserial_conv2d_nhwc_tcd_group(convs, 2, 1)
    for o, (act, wt, L) in zip(outs, samples):
        for img in (0, 97, 255):
            ref = oracle.conv2d_nhwc_enc(act[img:img + 1].numpy(), 2, 0, wt.numpy(), 1, 1, stride=(L.s, L.s),
                                         pad=(L.pad, L.pad))
            np.testing.assert_array_equal(o[img:img + 1].cpu().numpy(), ref, err_msg=f"layer {L.name} image {img}")


def test_conv_tcd_rejects():
    """Validation before launch: geometry the TMA im2col mode cannot encode, the FP4 bound,
    unsupported precisions; nothing written."""
    out = torch.full((1, 4, 4, 8), -7, dtype=torch.int32, device=DEV)
    ad = torch.zeros((1, 16, 32), dtype=torch.uint8, device=DEV)
    wd = torch.zeros((1 * 8 * 9 * 32,), dtype=torch.uint8, device=DEV)
    with pytest.raises(bs.BitserialError, match="stride"):
        bs.bitserial_conv2d_nhwc_tcd(ad, 2, wd, 1, 1, 4, 4, 8, 8, 3, 3, 9, 1, out=out)
    with pytest.raises(bs.BitserialError, match="a_bits"):
        bs.bitserial_conv2d_nhwc_tcd(ad, 5, wd, 1, 1, 4, 4, 8, 8, 3, 3, 1, 1, out=out)
    with pytest.raises(bs.BitserialError, match="2\\^22"):
        bs.bitserial_conv2d_nhwc_tcd(ad, 4, wd, 4, 1, 4, 4, 20000, 8, 3, 3, 1, 1, out=out)
    torch.cuda.synchronize()
    assert bool((out == -7).all())


# ------------------------------------------------------------------ dense
DENSE_SHAPES = [(1, 1, 1), (1, 7, 33), (3, 5, 100), (129, 65, 250), (300, 200, 576), (64, 256, 4096),
                (257, 130, 1000), (5, 1000, 129), (1000, 512, 96), (128, 128, 256), (300, 1500, 1000),
                (129, 1024, 520)]


@pytest.mark.parametrize("m,n,k", DENSE_SHAPES)
@pytest.mark.parametrize("a_bits,w_bits", [(1, 1), (2, 1), (2, 2), (4, 1), (4, 2), (3, 3)])
def test_dense_tcd_parity(m, n, k, a_bits, w_bits):
    for w_enc in (bs.UNIPOLAR, bs.BIPOLAR):
        a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=m * 31 + n * 7 + k + 3 * a_bits + w_bits + w_enc)
        ref = oracle.dense_enc(a.numpy(), a_bits, 0, w.numpy(), w_bits, w_enc)
        ad = bs.digitpack(a.to(DEV), a_bits)
        wd = bs.dense_tcd_prepare_weights(bs.bitpack(w.to(DEV), w_bits), w_bits, w_enc, n, k)
        got = bs.bitserial_dense_tcd(ad, a_bits, wd, w_bits, m, n, k, w_enc=w_enc)
        np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"{m}x{n}x{k} A{a_bits}W{w_bits} {w_enc}")


@pytest.mark.parametrize("a_enc,w_enc", ENC_PAIRS)
def test_dense_tcd_encodings(a_enc, w_enc):
    for (m, n, k, a_bits, w_bits) in ((130, 72, 100, 2, 1), (257, 132, 1000, 3, 2), (64, 256, 4096, 1, 1)):
        a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=a_enc * 100 + w_enc * 10 + a_bits + k)
        ref = oracle.dense_enc(a.numpy(), a_bits, a_enc, w.numpy(), w_bits, w_enc)
        ad = bs.digitpack(a.to(DEV), a_bits, a_enc)
        wd = bs.dense_tcd_prepare_weights(bs.bitpack(w.to(DEV), w_bits), w_bits, w_enc, n, k)
        got = bs.bitserial_dense_tcd(ad, a_bits, wd, w_bits, m, n, k, a_enc=a_enc, w_enc=w_enc)
        np.testing.assert_array_equal(got.cpu().numpy(), ref)


def _near_max_codes(rows, k, g, base, alts, p_alt=0.002):
    x = torch.full((rows, k), base, dtype=torch.uint8)
    sel = torch.rand((rows, k), generator=g) < p_alt
    pick = torch.randint(0, len(alts), (rows, k), generator=g)
    return torch.where(sel, torch.tensor(alts, dtype=torch.uint8)[pick], x)


# (a_bits, a_enc, w_bits, w_enc, K): K * max|a| * max|w| just under the FP4 bound 2^22
FP4_BOUND_CASES = [
    (1, 0, 1, 0, 4_194_303), (1, 0, 1, 1, 4_194_303), (4, 0, 4, 0, 18_641), (4, 0, 4, 1, 18_641),
    (4, 2, 4, 2, 65_535), (2, 1, 2, 1, 466_033),
]


@pytest.mark.parametrize("a_bits,a_enc,w_bits,w_enc,k", FP4_BOUND_CASES)
def test_dense_tcd_at_fp4_bound(a_bits, a_enc, w_bits, w_enc, k):
    """The digit path's FP32 accumulation exact at the ABI bound (near-max codes with a sparse
    sprinkle of other codes: odd low bits on a running sum near 2^22)."""
    m, n = 5, 9
    g = inputs.gen(k * 31 + a_bits * 7 + w_bits + 100 * a_enc + 1000 * w_enc)
    a_max = (1 << a_bits) - 1 if a_enc != 2 else 1 << (a_bits - 1)
    w_max = (1 << w_bits) - 1 if w_enc != 2 else 1 << (w_bits - 1)
    a = _near_max_codes(m, k, g, a_max, [0, 1, (1 << a_bits) - 1] + ([9, 11, 15] if a_enc == 2 else []))
    w = _near_max_codes(n, k, g, w_max, [0, 1] + ([9, 11, 15] if w_enc == 2 else []))
    w[n - 1] = 0 if w_enc == 1 else w_max
    ref = oracle.dense_enc(a.numpy(), a_bits, a_enc, w.numpy(), w_bits, w_enc)
    bound = k * (a_max if a_enc != 1 else (1 << a_bits) - 1) * (w_max if w_enc != 1 else (1 << w_bits) - 1)
    assert bound < 1 << 22 and int(np.abs(ref).max()) > 0.99 * bound
    ad = bs.digitpack(a.to(DEV), a_bits, a_enc)
    wd = bs.dense_tcd_prepare_weights(bs.bitpack(w.to(DEV), w_bits), w_bits, w_enc, n, k)
    got = bs.bitserial_dense_tcd(ad, a_bits, wd, w_bits, m, n, k, a_enc=a_enc, w_enc=w_enc)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("size,a_bits,w_bits", [(4096, 2, 1), (8192, 1, 1), (8192, 4, 2), (16384, 2, 1)])
def test_dense_tcd_gemm_sweep_sampled(size, a_bits, w_bits):
    """BASELINE configs[4] at full size on the digit path: 64 rows spread over C plus the first
    and last rows against the oracle."""
    m = n = k = size
    g = inputs.gen(size + 10 * a_bits + w_bits)
    a = inputs.codes((m, k), a_bits, g)
    w = inputs.codes((n, k), w_bits, g)
    ad = bs.digitpack(a.to(DEV), a_bits)
    wd = bs.dense_tcd_prepare_weights(bs.bitpack(w.to(DEV), w_bits), w_bits, bs.BIPOLAR, n, k)
    got = bs.bitserial_dense_tcd(ad, a_bits, wd, w_bits, m, n, k, w_enc=bs.BIPOLAR)
    rows = sorted(set([0, m - 1] + list(range(7, m, m // 64))))
    ref = oracle.dense_enc(a[rows].numpy(), a_bits, 0, w.numpy(), w_bits, bs.BIPOLAR)
    np.testing.assert_array_equal(got[rows].cpu().numpy(), ref)


@pytest.fixture
def tuning():
    used = []

    def set_(knob, value):
        bs.set_tuning(knob, value)
        used.append(knob)
    yield set_
    for k in used:
        bs.set_tuning(k, 0)


@pytest.mark.parametrize("a_src", [1, 2])
@pytest.mark.parametrize("b_stream", [0, 1])
@pytest.mark.parametrize("a_bits,w_bits", [(2, 1), (4, 2), (1, 3)])
def test_conv_tcd_operand_sources(tuning, a_src, b_stream, a_bits, w_bits):
    """Every conv case with the activations gathered by TMA im2col (1) or by the cp.async
    producer warps (2), and the weights resident per N block or streamed per stage."""
    tuning(bs.TUNE_TCD_A_SRC, a_src)
    tuning(bs.TUNE_TCD_B_STREAM, b_stream)
    for case in CONV_CASES:
        n, h, w, c, oc, kh, kw, s, p = case
        g = inputs.gen(n * 1000 + h * 37 + c * 7 + oc + 11 * a_bits + w_bits + 5 * a_src + b_stream)
        act = inputs.codes((n, h, w, c), a_bits, g)
        wt = inputs.codes((oc, kh, kw, c), w_bits, g)
        ref = oracle.conv2d_nhwc_enc(act.numpy(), a_bits, 0, wt.numpy(), w_bits, 1, stride=(s, s), pad=(p, p))
        got = run_conv(act, a_bits, 0, wt, w_bits, 1, s, p)
        np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"{case} a_src={a_src} b_stream={b_stream}")


@pytest.mark.parametrize("mcast_off", [2, 1])
@pytest.mark.parametrize("m,n,k,a_bits,w_bits", [(512, 1024, 4096, 2, 1), (256, 1000, 2000, 2, 2), (384, 2048, 1500, 4, 1),
                                                 (258, 1030, 2600, 1, 3)])
def test_dense_tcd_cluster_multicast(tuning, mcast_off, m, n, k, a_bits, w_bits):
    """Dense products with streamed weights: 2-CTA clusters that each load half of every weight
    chunk and multicast it to both (knob 2), and the same without the clusters (knob 1); ragged N."""
    tuning(bs.TUNE_TCD_MCAST, mcast_off)
    for w_enc in (bs.UNIPOLAR, bs.BIPOLAR):
        a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=m + n + k + a_bits + w_bits + w_enc)
        ref = oracle.dense_enc(a.numpy(), a_bits, 0, w.numpy(), w_bits, w_enc)
        ad = bs.digitpack(a.to(DEV), a_bits)
        wd = bs.dense_tcd_prepare_weights(bs.bitpack(w.to(DEV), w_bits), w_bits, w_enc, n, k)
        got = bs.bitserial_dense_tcd(ad, a_bits, wd, w_bits, m, n, k, w_enc=w_enc)
        np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"{m}x{n}x{k} mcast_off={mcast_off}")
