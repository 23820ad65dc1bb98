"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle,
element by element, bit-exact (int32, zero tolerance: the method computes an exact
integer result, DESIGN.md §3 R14).  Inputs come from paper_1810_11066_b200.inputs
(seeded, uniform codes); expected values only ever come from oracle/."""
import numpy as np
import pytest
import torch

import oracle
import paper_1810_11066_b200 as bs
from paper_1810_11066_b200 import inputs

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture
def tuning():
    """Set bs_set_tuning knobs for one test; every knob set is reset to 0 afterwards."""
    used = []

    def set_(knob, value):
        bs.set_tuning(knob, value)
        used.append(knob)
    yield set_
    for k in used:
        bs.set_tuning(k, 0)


def enc(bipolar):
    return bs.BIPOLAR if bipolar else bs.UNIPOLAR


def gpu_pack(x_cpu, bits):
    return bs.bitpack(x_cpu.to(DEV), bits)


# ----------------------------------------------------------------------- bitpack
@pytest.mark.parametrize("rows,k,bits", [(1, 1, 1), (3, 31, 2), (5, 32, 1), (7, 33, 3), (4, 100, 4),
                                         (9, 64, 2), (2, 130, 8), (3136, 64, 2), (513, 4096, 2),
                                         (1000, 48, 5), (37, 3, 2), (11, 576, 7)])
def test_bitpack_parity(rows, k, bits):
    g = inputs.gen(rows * 7919 + k * 31 + bits)
    x = inputs.codes((rows, k), bits, g)
    got = gpu_pack(x, bits).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(got, oracle.bitpack(x.numpy(), bits))


def test_bitpack_unaligned_source():
    g = inputs.gen(5)
    big = inputs.codes((4 * 64 + 16,), 2, g).to(DEV)
    x = big[16:].view(4, 64)            # 16-byte aligned but offset view
    got = bs.bitpack(x.contiguous(), 2).cpu().numpy().view(np.uint32)
    np.testing.assert_array_equal(got, oracle.bitpack(x.cpu().numpy(), 2))


# ------------------------------------------------------------------------- dense
DENSE_SHAPES = [(1, 1, 1), (1, 7, 33), (3, 5, 100), (8, 64, 64), (129, 65, 250),
                (300, 200, 576), (64, 256, 4096), (257, 130, 1000), (1, 4096, 4096), (5, 1000, 129)]
PRECISIONS = [(1, 1), (2, 1), (2, 2), (4, 1), (4, 2), (1, 2), (3, 3), (4, 4), (5, 1), (8, 1), (2, 6)]


@pytest.mark.parametrize("m,n,k", DENSE_SHAPES)
@pytest.mark.parametrize("a_bits,w_bits", [(1, 1), (2, 1), (2, 2)])
@pytest.mark.parametrize("bipolar", [False, True])
def test_dense_parity_auto(m, n, k, a_bits, w_bits, bipolar):
    a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=m * 1000 + n + k + a_bits)
    ref = oracle.dense(a.numpy(), a_bits, w.numpy(), w_bits, bipolar)
    got = bs.bitserial_dense(gpu_pack(a, a_bits), a_bits, gpu_pack(w, w_bits), w_bits, enc(bipolar), m, n, k)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("algo", [bs.ALGO_POPC, bs.ALGO_POPC_LIT])
@pytest.mark.parametrize("a_bits,w_bits", PRECISIONS)
@pytest.mark.parametrize("bipolar", [False, True])
def test_dense_parity_tiled_all_precisions(algo, a_bits, w_bits, bipolar):
    m, n, k = 150, 77, 300
    a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=10 * a_bits + w_bits)
    ref = oracle.dense(a.numpy(), a_bits, w.numpy(), w_bits, bipolar)
    got = bs.bitserial_dense(gpu_pack(a, a_bits), a_bits, gpu_pack(w, w_bits), w_bits, enc(bipolar), m, n, k,
                             algo=algo)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("m", [1, 2, 5, 8])
@pytest.mark.parametrize("a_bits,w_bits", [(1, 1), (2, 1), (2, 2), (4, 1), (4, 2), (1, 2)])
@pytest.mark.parametrize("k", [64, 100, 4096])
def test_gemv_parity(m, a_bits, w_bits, k):
    n = 300
    for bipolar in (False, True):
        a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=m + k + a_bits * 10 + w_bits)
        ref = oracle.dense(a.numpy(), a_bits, w.numpy(), w_bits, bipolar)
        got = bs.bitserial_dense(gpu_pack(a, a_bits), a_bits, gpu_pack(w, w_bits), w_bits, enc(bipolar), m, n, k,
                                 algo=bs.ALGO_GEMV)
        np.testing.assert_array_equal(got.cpu().numpy(), ref)
        got = bs.bitserial_dense_i8(a.to(DEV), a_bits, gpu_pack(w, w_bits), w_bits, enc(bipolar), n)
        np.testing.assert_array_equal(got.cpu().numpy(), ref)


def test_dense_i8_tiled_path():
    m, n, k = 100, 64, 200
    a, w = inputs.dense_operands(m, n, k, 2, 1, seed=3)
    ref = oracle.dense(a.numpy(), 2, w.numpy(), 1, True)
    got = bs.bitserial_dense_i8(a.to(DEV), 2, gpu_pack(w, 1), 1, bs.BIPOLAR, n)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


# -------------------------------------------------------------------------- conv
CONV_CASES = [
    # n, h, w, c, oc, kh, kw, sh, sw, ph, pw
    (1, 9, 7, 5, 3, 3, 3, 1, 1, 1, 1),
    (2, 8, 11, 33, 20, 3, 3, 2, 2, 1, 1),
    (3, 6, 5, 64, 70, 1, 1, 2, 2, 0, 0),
    (1, 7, 7, 3, 5, 3, 2, 1, 2, 0, 1),
    (2, 5, 9, 17, 6, 2, 3, 3, 1, 2, 0),
    (1, 13, 13, 128, 129, 3, 3, 1, 1, 1, 1),
    (2, 7, 7, 512, 64, 3, 3, 1, 1, 1, 1),
    (1, 15, 15, 256, 130, 3, 3, 2, 2, 1, 1),
    (4, 1, 1, 64, 8, 1, 1, 1, 1, 0, 0),
    (1, 3, 3, 64, 4, 5, 5, 1, 1, 2, 2),   # kernel larger than image with pad
]


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("a_bits,w_bits", [(1, 1), (2, 1), (2, 2), (4, 2), (3, 1)])
@pytest.mark.parametrize("bipolar", [False, True])
def test_conv_parity(case, a_bits, w_bits, bipolar):
    n, h, w, c, oc, kh, kw, sh, sw, ph, pw = case
    g = inputs.gen(sum(case) * 100 + a_bits * 10 + w_bits)
    act = inputs.codes((n, h, w, c), a_bits, g)
    wt = inputs.codes((oc, kh, kw, c), w_bits, g)
    ref = oracle.conv2d_nhwc(act.numpy(), a_bits, wt.numpy(), w_bits, bipolar, stride=(sh, sw), pad=(ph, pw))
    wp = gpu_pack(wt.view(oc * kh * kw, c), w_bits)
    for algo in (bs.ALGO_POPC, bs.ALGO_POPC_LIT):
        got = bs.bitserial_conv2d_nhwc(gpu_pack(act.view(-1, c), a_bits), a_bits, wp, w_bits, enc(bipolar),
                                       n, h, w, c, oc, kh, kw, (sh, sw), (ph, pw), algo=algo)
        np.testing.assert_array_equal(got.cpu().numpy(), ref)
    got = bs.bitserial_conv2d_nhwc_i8(act.to(DEV), a_bits, wp, w_bits, enc(bipolar), oc, kh, kw, (sh, sw), (ph, pw))
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


def _layer_run(L, batch, a_bits, w_bits, bipolar, seed):
    act, wt = inputs.conv_operands(L, batch, a_bits, w_bits, seed)
    wp = gpu_pack(wt.view(L.oc * L.k * L.k, L.ic), w_bits)
    got = bs.bitserial_conv2d_nhwc_i8(act.to(DEV), a_bits, wp, w_bits, enc(bipolar), L.oc, L.k, L.k, L.s, L.pad)
    return act, wt, got


def test_config1_conv_l2_batch1_full():
    """BASELINE configs[0]: 56x56x64 -> 64, 3x3 s1 p1, A2W1 bipolar, batch 1 — full compare."""
    L = inputs.TABLE1[2]
    act, wt, got = _layer_run(L, 1, 2, 1, True, inputs.seed_for(1, 2, 1, "bipolar", 2))
    ref = oracle.conv2d_nhwc(act.numpy(), 2, wt.numpy(), 1, True, stride=(1, 1), pad=(1, 1))
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


def test_config2_gemv_full():
    """BASELINE configs[1]: K = N = 4096, A2W1 bipolar, batch 1 — full compare, fused path."""
    a, w = inputs.dense_operands(1, 4096, 4096, 2, 1, inputs.seed_for(2, 2, 1, "bipolar"))
    ref = oracle.dense(a.numpy(), 2, w.numpy(), 1, True)
    got = bs.bitserial_dense_i8(a.to(DEV), 2, gpu_pack(w, 1), 1, bs.BIPOLAR, 4096)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("layer", inputs.BASELINE_LAYERS + (3,))
def test_config3_resnet_layers_batch1_full(layer):
    """BASELINE configs[2]: every layer x {A1W1, A2W1, A2W2} x {uni, bip}, batch 1, full compare."""
    L = inputs.TABLE1[layer]
    for (a_bits, w_bits) in [(1, 1), (2, 1), (2, 2)]:
        for bipolar in (False, True):
            e = "bipolar" if bipolar else "unipolar"
            act, wt, got = _layer_run(L, 1, a_bits, w_bits, bipolar, inputs.seed_for(3, a_bits, w_bits, e, layer))
            ref = oracle.conv2d_nhwc(act.numpy(), a_bits, wt.numpy(), w_bits, bipolar,
                                     stride=(L.s, L.s), pad=(L.pad, L.pad))
            np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"L{layer} A{a_bits}W{w_bits} {e}")


@pytest.mark.parametrize("layer", inputs.BASELINE_LAYERS)
def test_config4_batch256_sampled_images(layer):
    """BASELINE configs[3]: batch 256, A2W1 bipolar, in the bench's launch configuration
    (whole batch in one call); the oracle checks images 0, 131 and 255 in full."""
    L = inputs.TABLE1[layer]
    act, wt, got = _layer_run(L, 256, 2, 1, True, inputs.seed_for(4, 2, 1, "bipolar", layer))
    got = got.cpu().numpy()
    for img in (0, 131, 255):
        ref = oracle.conv2d_nhwc(act[img:img + 1].numpy(), 2, wt.numpy(), 1, True,
                                 stride=(L.s, L.s), pad=(L.pad, L.pad))
        np.testing.assert_array_equal(got[img:img + 1], ref, err_msg=f"L{layer} image {img}")


@pytest.mark.parametrize("size", [4096, 8192, 16384])
@pytest.mark.parametrize("a_bits,w_bits,bipolar", [(1, 1, False), (2, 1, True), (4, 2, True)])
def test_config5_gemm_sampled_rows(size, a_bits, w_bits, bipolar):
    """BASELINE configs[4]: M = N = K GEMM; full GPU product, oracle on sampled rows."""
    e = "bipolar" if bipolar else "unipolar"
    a, w = inputs.dense_operands(size, size, size, a_bits, w_bits, inputs.seed_for(5, a_bits, w_bits, e))
    wp = gpu_pack(w, w_bits)
    got = bs.bitserial_dense_i8(a.to(DEV), a_bits, wp, w_bits, enc(bipolar), size)
    rows = [0, 1, size // 2 + 3, size - 1]
    ref = oracle.dense(a[rows].numpy(), a_bits, w.numpy(), w_bits, bipolar)
    np.testing.assert_array_equal(got[rows].cpu().numpy(), ref)


# ---------------------------------------------------------------- invariants / edges
def test_bipolar_identity_and_literal_agree_on_gpu():
    m, n, k = 200, 96, 1000
    a, w = inputs.dense_operands(m, n, k, 2, 2, seed=77)
    ap, wp = gpu_pack(a, 2), gpu_pack(w, 2)
    uni = bs.bitserial_dense(ap, 2, wp, 2, bs.UNIPOLAR, m, n, k).long()
    bip = bs.bitserial_dense(ap, 2, wp, 2, bs.BIPOLAR, m, n, k, algo=bs.ALGO_POPC).long()
    lit = bs.bitserial_dense(ap, 2, wp, 2, bs.BIPOLAR, m, n, k, algo=bs.ALGO_POPC_LIT).long()
    s = a.long().sum(1, keepdim=True).to(DEV)
    assert torch.equal(bip, lit)
    assert torch.equal(bip, 2 * uni - 3 * s)


def test_extreme_values_max_bits():
    """All-max codes at the accumulator bound region: A8W1 with K = 8000 (255*8000 < 2^31)."""
    m, n, k = 3, 40, 8000
    a = torch.full((m, k), 255, dtype=torch.uint8)
    w = torch.ones((n, k), dtype=torch.uint8)
    ref = oracle.dense(a.numpy(), 8, w.numpy(), 1, False)
    got = bs.bitserial_dense(gpu_pack(a, 8), 8, gpu_pack(w, 1), 1, bs.UNIPOLAR, m, n, k, algo=bs.ALGO_POPC)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)
    assert int(ref[0, 0]) == 255 * 8000


def test_errors_surface_as_exceptions():
    x = torch.zeros(4, 32, dtype=torch.uint8, device=DEV)
    with pytest.raises(bs.BitserialError, match="BS_ERR_INVALID_ARG"):
        bs.bitpack(x, 9)
    p = bs.bitpack(x, 2)
    with pytest.raises(bs.BitserialError, match="BS_ERR_SHAPE"):
        bs.bitserial_conv2d_nhwc(p, 2, p, 2, bs.UNIPOLAR, 1, 2, 2, 32, 4, 3, 3, 1, 0)


def test_host_e2e_entry():
    L = inputs.TABLE1[9]
    act, wt = inputs.conv_operands(L, 2, 2, 1, seed=9)
    wp = gpu_pack(wt.view(L.oc * 9, L.ic), 1)
    oh = bs.conv_out_extent(L.h, 3, 1, 1)
    out_host = torch.empty((2, oh, oh, L.oc), dtype=torch.int32).pin_memory()
    act_host = act.pin_memory()
    act_dev = torch.empty_like(act, device=DEV)
    out_dev = torch.empty_like(out_host, device=DEV)
    ws = torch.empty(bs.conv2d_workspace_bytes(2, L.h, L.w, L.ic, 2), dtype=torch.uint8, device=DEV)
    bs.bitserial_conv2d_nhwc_host(act_host, 2, wp, 1, bs.BIPOLAR, L.oc, 3, 3, 1, 1, out_host, act_dev, out_dev, ws)
    ref = oracle.conv2d_nhwc(act.numpy(), 2, wt.numpy(), 1, True, stride=(1, 1), pad=(1, 1))
    np.testing.assert_array_equal(out_host.numpy(), ref)


@pytest.mark.parametrize("a_bits", [1, 2, 3, 4])
@pytest.mark.parametrize("w_bits", [1, 2, 3, 4])
def test_limit_study_grid_parity(a_bits, w_bits):
    """layer 9 at every A, W in 1..4, both encodings,
    batch 2 — the kernels the limit study times — full compare."""
    L = inputs.TABLE1[9]
    for bipolar in (False, True):
        act, wt, got = _layer_run(L, 2, a_bits, w_bits, bipolar, seed=7 * a_bits + w_bits + 100 * bipolar)
        ref = oracle.conv2d_nhwc(act.numpy(), a_bits, wt.numpy(), w_bits, bipolar, stride=(1, 1), pad=(1, 1))
        np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"A{a_bits}W{w_bits} bipolar={bipolar}")


@pytest.mark.parametrize("case", [(1, 4, 4, 600, 40, 3, 3, 1, 1, 1, 1), (1, 7, 7, 512, 512, 3, 3, 1, 1, 1, 1),
                                  (2, 14, 14, 256, 512, 1, 1, 2, 2, 0, 0), (1, 2, 3, 2048, 16, 1, 3, 1, 1, 0, 1)])
def test_split_k_small_mn(case):
    """Small M x N with long K takes the split-K path (int32 atomics into a zeroed
    output); exact regardless of the order partials land."""
    n, h, w, c, oc, kh, kw, sh, sw, ph, pw = case
    g = inputs.gen(sum(case))
    act = inputs.codes((n, h, w, c), 2, g)
    wt = inputs.codes((oc, kh, kw, c), 1, g)
    ref = oracle.conv2d_nhwc(act.numpy(), 2, wt.numpy(), 1, True, stride=(sh, sw), pad=(ph, pw))
    wp = gpu_pack(wt.view(oc * kh * kw, c), 1)
    for _ in range(3):
        got = bs.bitserial_conv2d_nhwc_i8(act.to(DEV), 2, wp, 1, bs.BIPOLAR, oc, kh, kw, (sh, sw), (ph, pw))
        np.testing.assert_array_equal(got.cpu().numpy(), ref)


# ------------------------------------------------------------ tensor-core path
TC_PRECISIONS = [(1, 1), (2, 1), (2, 2), (1, 2), (3, 1), (3, 2), (4, 1), (4, 2),
                 (1, 3), (2, 3), (3, 3), (4, 3), (1, 4), (2, 4), (3, 4), (4, 4)]


@pytest.mark.parametrize("a_bits,w_bits", TC_PRECISIONS)
@pytest.mark.parametrize("bipolar", [False, True])
@pytest.mark.parametrize("m,n,k", [(1, 16, 32), (130, 64, 200), (257, 130, 1000), (128, 256, 4096), (300, 300, 33)])
def test_dense_tc_parity(a_bits, w_bits, bipolar, m, n, k):
    a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=31 * a_bits + w_bits + m + k)
    ref = oracle.dense(a.numpy(), a_bits, w.numpy(), w_bits, bipolar)
    got = bs.bitserial_dense_tc(gpu_pack(a, a_bits), a_bits, gpu_pack(w, w_bits), w_bits, enc(bipolar), m, n, k)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("a_bits,w_bits", [(1, 1), (2, 1), (2, 2), (4, 2)])
@pytest.mark.parametrize("bipolar", [False, True])
def test_conv_tc_parity(case, a_bits, w_bits, bipolar):
    n, h, w, c, oc, kh, kw, sh, sw, ph, pw = case
    g = inputs.gen(sum(case) * 100 + a_bits * 10 + w_bits + 5)
    act = inputs.codes((n, h, w, c), a_bits, g)
    wt = inputs.codes((oc, kh, kw, c), w_bits, g)
    ref = oracle.conv2d_nhwc(act.numpy(), a_bits, wt.numpy(), w_bits, bipolar, stride=(sh, sw), pad=(ph, pw))
    wp = gpu_pack(wt.view(oc * kh * kw, c), w_bits)
    got = bs.bitserial_conv2d_nhwc_tc(gpu_pack(act.view(-1, c), a_bits), a_bits, wp, w_bits, enc(bipolar),
                                      n, h, w, c, oc, kh, kw, (sh, sw), (ph, pw))
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("layer", inputs.BASELINE_LAYERS)
def test_conv_tc_resnet_layers(layer):
    """TC path on every BASELINE layer, batch 2, A2W1 bipolar and A2W2 unipolar, full compare."""
    L = inputs.TABLE1[layer]
    for a_bits, w_bits, bipolar in ((2, 1, True), (2, 2, False)):
        act, wt = inputs.conv_operands(L, 2, a_bits, w_bits, seed=layer + 11 * a_bits + w_bits)
        wp = gpu_pack(wt.view(L.oc * L.k * L.k, L.ic), w_bits)
        got = bs.bitserial_conv2d_nhwc_tc(gpu_pack(act.view(-1, L.ic), a_bits), a_bits, wp, w_bits, enc(bipolar),
                                          2, L.h, L.w, L.ic, L.oc, L.k, L.k, L.s, L.pad)
        ref = oracle.conv2d_nhwc(act.numpy(), a_bits, wt.numpy(), w_bits, bipolar, stride=(L.s, L.s),
                                 pad=(L.pad, L.pad))
        np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"L{layer} A{a_bits}W{w_bits}")


# ------------------------------------------- tensor-core path, prepared weights
TC_FORMATS = [bs.TC_I8, bs.TC_F4]


def _tc_conv_prepared(act, a_bits, wt, w_bits, bipolar, stride, pad, fused, fmt=bs.TC_DEFAULT):
    n, h, w, c = act.shape
    oc, kh, kw, _ = wt.shape
    wp = gpu_pack(wt.reshape(oc * kh * kw, c), w_bits)
    w_tc = bs.conv2d_tc_prepare_weights(wp, w_bits, enc(bipolar), oc, kh, kw, c, tc_format=fmt)
    if fused:
        return bs.bitserial_conv2d_nhwc_tc_i8(act.to(DEV), a_bits, w_tc, w_bits, oc, kh, kw, stride, pad,
                                              tc_format=fmt)
    return bs.bitserial_conv2d_nhwc_tc_prepared(gpu_pack(act.reshape(-1, c), a_bits), a_bits, w_tc, w_bits,
                                                n, h, w, c, oc, kh, kw, stride, pad, tc_format=fmt)


@pytest.mark.parametrize("fmt", TC_FORMATS)
@pytest.mark.parametrize("bn", ["64", "128"])
@pytest.mark.parametrize("a_bits,w_bits", TC_PRECISIONS)
@pytest.mark.parametrize("bipolar", [False, True])
def test_conv_tc_every_tile_width(tuning, fmt, bn, a_bits, w_bits, bipolar):
    """Each compiled tile width (BS_TUNE_TC_TILE_N forces it; configurations that do not fit shared
    memory fall back to a narrower one) on a ragged case: M = 2*13*11 = 286 (3 row tiles,
    tail 30), OC = 300 (ragged column tiles, OC % 4 = 0 so the TMA-store epilogue runs),
    K = 9 taps x 4 words (9 K chunks)."""
    tuning(bs.TUNE_TC_TILE_N, int(bn))
    g = inputs.gen(int(bn) + 10 * a_bits + w_bits + (100 if bipolar else 0))
    act = inputs.codes((2, 13, 11, 96), a_bits, g)
    wt = inputs.codes((300, 3, 3, 96), w_bits, g)
    ref = oracle.conv2d_nhwc(act.numpy(), a_bits, wt.numpy(), w_bits, bipolar, stride=(1, 1), pad=(1, 1))
    got = _tc_conv_prepared(act, a_bits, wt, w_bits, bipolar, 1, 1, fused=True, fmt=fmt)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("fmt", TC_FORMATS)
@pytest.mark.parametrize("slots", [0, 2, 3])
@pytest.mark.parametrize("epi", [0, 1])
@pytest.mark.parametrize("a_bits,w_bits,bipolar", [(2, 1, True), (1, 2, False), (4, 2, True)])
@pytest.mark.parametrize("oc", [64, 100, 128, 300])
def test_conv_tc_b_modes(tuning, fmt, slots, epi, a_bits, w_bits, bipolar, oc):
    """Weights resident in the shared-memory chunk slots (all K chunks fit: loaded once per
    N block, reused by the CTA's next tiles of that block) versus streamed through a ring of
    2 or 3 slots (BS_TUNE_TC_B_SLOTS; fewer slots than the 5 / 9 K chunks), with 1..3 N
    blocks, and the direct-store versus TMA-store epilogue, on a ragged 3x3 s2 case
    (M = 3*10*10 = 300: 3 row tiles; K = 9 taps x 2 words)."""
    if slots:
        tuning(bs.TUNE_TC_B_SLOTS, slots)
    tuning(bs.TUNE_TC_EPILOGUE, epi)
    g = inputs.gen(oc + 10 * a_bits + w_bits)
    act = inputs.codes((3, 19, 20, 64), a_bits, g)
    wt = inputs.codes((oc, 3, 3, 64), w_bits, g)
    ref = oracle.conv2d_nhwc(act.numpy(), a_bits, wt.numpy(), w_bits, bipolar, stride=(2, 2), pad=(1, 1))
    got = _tc_conv_prepared(act, a_bits, wt, w_bits, bipolar, 2, 1, fused=True, fmt=fmt)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("fmt", TC_FORMATS)
@pytest.mark.parametrize("case", CONV_CASES)
@pytest.mark.parametrize("fused", [False, True])
def test_conv_tc_prepared_cases(fmt, case, fused):
    """Prepared-weight entries (with and without in-call packing) on the ragged /
    odd-geometry cases, including OC % 4 != 0 (plain-store epilogue) and K tails."""
    n, h, w, c, oc, kh, kw, sh, sw, ph, pw = case
    for a_bits, w_bits, bipolar in ((2, 1, True), (3, 2, False)):
        g = inputs.gen(sum(case) * 7 + a_bits + 3 * w_bits)
        act = inputs.codes((n, h, w, c), a_bits, g)
        wt = inputs.codes((oc, kh, kw, c), w_bits, g)
        ref = oracle.conv2d_nhwc(act.numpy(), a_bits, wt.numpy(), w_bits, bipolar, stride=(sh, sw), pad=(ph, pw))
        got = _tc_conv_prepared(act, a_bits, wt, w_bits, bipolar, (sh, sw), (ph, pw), fused, fmt)
        np.testing.assert_array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("fmt", TC_FORMATS)
@pytest.mark.parametrize("m,n,k", [(1, 16, 32), (130, 64, 200), (257, 132, 1000), (384, 512, 4096), (300, 300, 33)])
@pytest.mark.parametrize("a_bits,w_bits,bipolar", [(1, 1, False), (2, 1, True), (4, 2, True), (3, 2, False)])
def test_dense_tc_prepared(fmt, m, n, k, a_bits, w_bits, bipolar):
    a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=17 * a_bits + w_bits + m + n + k)
    ref = oracle.dense(a.numpy(), a_bits, w.numpy(), w_bits, bipolar)
    w_tc = bs.dense_tc_prepare_weights(gpu_pack(w, w_bits), w_bits, enc(bipolar), n, k, tc_format=fmt)
    got = bs.bitserial_dense_tc_i8(a.to(DEV), a_bits, w_tc, w_bits, n, tc_format=fmt)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)
    got2 = bs.bitserial_dense_tc_prepared(gpu_pack(a, a_bits), a_bits, w_tc, w_bits, m, n, k, tc_format=fmt)
    assert torch.equal(got, got2)


@pytest.mark.parametrize("fmt", TC_FORMATS)
@pytest.mark.parametrize("layer", inputs.BASELINE_LAYERS)
def test_config4_batch256_tc_sampled_images(fmt, layer):
    """BASELINE configs[3] in the bench's launch configuration on the tensor-core path
    (prepared weights, whole batch of 256 in one bs_bitserial_conv2d_nhwc_tc_i8 call,
    persistent kernel over every tile); the oracle checks images 0, 77, 200 and 255."""
    L = inputs.TABLE1[layer]
    act, wt = inputs.conv_operands(L, 256, 2, 1, inputs.seed_for(4, 2, 1, "bipolar", layer))
    got = _tc_conv_prepared(act, 2, wt, 1, True, L.s, L.pad, fused=True, fmt=fmt).cpu().numpy()
    for img in (0, 77, 200, 255):
        ref = oracle.conv2d_nhwc(act[img:img + 1].numpy(), 2, wt.numpy(), 1, True,
                                 stride=(L.s, L.s), pad=(L.pad, L.pad))
        np.testing.assert_array_equal(got[img:img + 1], ref, err_msg=f"L{layer} image {img}")


@pytest.mark.parametrize("fmt", TC_FORMATS)
def test_tc_repeated_calls_stable(fmt):
    """Persistent kernel re-launched back to back on one stream (as in the bench's CUDA
    graph): identical results every time (no stale TMEM / barrier state)."""
    L = inputs.TABLE1[6]
    act, wt = inputs.conv_operands(L, 8, 2, 1, seed=99)
    first = _tc_conv_prepared(act, 2, wt, 1, True, L.s, L.pad, fused=True, fmt=fmt)
    ref = oracle.conv2d_nhwc(act.numpy(), 2, wt.numpy(), 1, True, stride=(L.s, L.s), pad=(L.pad, L.pad))
    np.testing.assert_array_equal(first.cpu().numpy(), ref)
    for _ in range(5):
        assert torch.equal(_tc_conv_prepared(act, 2, wt, 1, True, L.s, L.pad, fused=True, fmt=fmt), first)


@pytest.mark.parametrize("fmt", TC_FORMATS)
@pytest.mark.parametrize("a_bits,w_bits", [(4, 2), (2, 2)])
def test_tc_accumulator_bound_extremes(fmt, a_bits, w_bits):
    """All-max codes on a long reduction: the largest |out| the configs reach
    (K * (2^A-1) * (2^W-1), BASELINE configs[4] A4W2 at K = 16384 -> 737,280) computed
    exactly by both formats (the FP4 path accumulates in FP32, exact below 2^24)."""
    m, n, k = 130, 72, 16384
    for bipolar in (False, True):
        a = torch.full((m, k), (1 << a_bits) - 1, dtype=torch.uint8)
        w = torch.full((n, k), (1 << w_bits) - 1, dtype=torch.uint8)
        w[1::2, ::3] = 0  # mixed signs / zeros in half the rows
        ref = oracle.dense(a.numpy(), a_bits, w.numpy(), w_bits, bipolar)
        w_tc = bs.dense_tc_prepare_weights(gpu_pack(w, w_bits), w_bits, enc(bipolar), n, k, tc_format=fmt)
        got = bs.bitserial_dense_tc_i8(a.to(DEV), a_bits, w_tc, w_bits, n, tc_format=fmt)
        np.testing.assert_array_equal(got.cpu().numpy(), ref)
    assert int(np.abs(ref).max()) == k * ((1 << a_bits) - 1) * ((1 << w_bits) - 1)


def _near_max_codes(rows, k, bits, g, base, alts, p_alt=0.002):
    """Codes equal to `base` except a sparse random sprinkle of the codes in `alts`
    (so sums sit just under the bound with odd, row-dependent low bits)."""
    x = torch.full((rows, k), base, dtype=torch.uint8)
    sel = torch.rand((rows, k), generator=g) < p_alt
    pick = torch.randint(0, len(alts), (rows, k), generator=g)
    alt = torch.tensor(alts, dtype=torch.uint8)[pick]
    return torch.where(sel, alt, x)


# (a_bits, a_enc, w_bits, w_enc, K): K * max|a| * max|w| just under the FP4 ABI bound
# 2^22 = 4,194,304 (abi.cu check_tc_bound) for every encoding family.
FP4_BOUND_CASES = [
    (1, 0, 1, 0, 4_194_303),   # A1W1: +1 increments on a running sum at 2^22 (FP32 ulp 0.5)
    (1, 0, 1, 1, 4_194_303),   # W1 bipolar: +-1
    (4, 0, 4, 0, 18_641),      # A4W4 unsigned x unipolar: 18,641 * 225 = 4,194,225
    (4, 0, 4, 1, 18_641),      # bipolar weights +-15
    (4, 2, 4, 2, 65_535),      # both signed: (-8)(-8) = 64 -> 4,194,240; signed-digit partials up to (11/8)^2 more
    (2, 1, 2, 1, 466_033),     # both bipolar (XNOR form): 466,033 * 9 = 4,194,297
]


@pytest.mark.parametrize("a_bits,a_enc,w_bits,w_enc,k", FP4_BOUND_CASES)
def test_tc_fp4_at_abi_bound(a_bits, a_enc, w_bits, w_enc, k):
    """The FP4 (kind::mxf4) format's exactness at its ABI bound: the dense product with
    K * max|a| * max|w| just below 2^22 (the largest magnitude check_tc_bound admits),
    near-max codes with a sparse sprinkle of other codes (odd low bits on a large running
    sum), against the oracle element by element.  The FP32 accumulator holds integers
    exactly below 2^24 (every digit product and partial sum is an integer,
    DESIGN.md R17/R21); this pins that the hardware's internal accumulation keeps them."""
    m, n = 5, 9
    g = inputs.gen(k * 31 + a_bits * 7 + w_bits + 100 * a_enc + 1000 * w_enc)
    a_max = (1 << a_bits) - 1 if a_enc != 2 else 1 << (a_bits - 1)      # code of the largest |value|
    w_max = (1 << w_bits) - 1 if w_enc != 2 else 1 << (w_bits - 1)
    a_alts = [0, 1, (1 << a_bits) - 1] + ([9, 11, 15] if a_enc == 2 else [])
    w_alts = [0, 1] + ([9, 11, 15] if w_enc == 2 else [])
    a = _near_max_codes(m, k, a_bits, g, a_max, a_alts)
    w = _near_max_codes(n, k, w_bits, g, w_max, w_alts)
    w[n - 1] = 0 if w_enc == 1 else w_max  # one weight row of constant sign: |sum| at its largest
    ref = oracle.dense_enc(a.numpy(), a_bits, a_enc, w.numpy(), w_bits, w_enc)
    bound = k * (a_max if a_enc != 1 else (1 << a_bits) - 1) * (w_max if w_enc != 1 else (1 << w_bits) - 1)
    assert bound < 1 << 22
    assert int(np.abs(ref).max()) > 0.99 * bound  # the case really sits at the bound
    w_tc = bs.dense_tc_prepare_weights(gpu_pack(w, w_bits), w_bits, w_enc, n, k, tc_format=bs.TC_F4)
    got = bs.bitserial_dense_tc_i8(a.to(DEV), a_bits, w_tc, w_bits, n, tc_format=bs.TC_F4, a_enc=a_enc, w_enc=w_enc)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


def test_tc_fp4_bound_rejects_past_2p22():
    """One past the bound is refused before launch (BS_ERR_OVERFLOW), nothing written."""
    k = 18_642  # 18,642 * 225 = 4,194,450 >= 2^22
    a = torch.full((2, k), 15, dtype=torch.uint8, device=DEV)
    w_tc = bs.dense_tc_prepare_weights(bs.bitpack(torch.full((3, k), 15, dtype=torch.uint8, device=DEV), 4), 4,
                                       bs.UNIPOLAR, 3, k, tc_format=bs.TC_F4)
    out = torch.full((2, 3), -7, dtype=torch.int32, device=DEV)
    with pytest.raises(bs.BitserialError, match="2\\^22"):
        bs.bitserial_dense_tc_i8(a, 4, w_tc, 4, 3, out=out, tc_format=bs.TC_F4)
    assert bool((out == -7).all())


@pytest.mark.parametrize("max_ctas", [1, 7, 148])
def test_bitpack_capped_grid(max_ctas):
    """bs_bitpack_ex with a small grid (the batched fast path plus its tail) packs
    exactly like the default launch."""
    for rows, k, bits in ((3136 * 4, 64, 2), (1001, 96, 3), (513, 4096, 1), (77, 100, 2)):
        g = inputs.gen(rows + k + bits + max_ctas)
        x = inputs.codes((rows, k), bits, g)
        got = bs.bitpack(x.to(DEV), bits, max_ctas=max_ctas).cpu().numpy().view(np.uint32)
        np.testing.assert_array_equal(got, oracle.bitpack(x.numpy(), bits))


# --------------------------------------- encodings on the tensor-core path (8f3)
ENC_PAIRS = [(a, w) for a in (bs.A_UNSIGNED, bs.A_BIPOLAR, bs.A_SIGNED) for w in (bs.UNIPOLAR, bs.BIPOLAR, bs.SIGNED)]


@pytest.mark.parametrize("a_enc,w_enc", ENC_PAIRS)
@pytest.mark.parametrize("a_bits,w_bits", [(1, 1), (2, 1), (2, 2), (3, 2), (4, 3), (1, 4)])
def test_conv_tc_encodings(a_enc, w_enc, a_bits, w_bits):
    """FP4 tensor-core conv with every (activation, weight) encoding — bipolar x bipolar
    is the XNOR form of PAPER.md:503, signed the sign-weighted Eq. 2 of PAPER.md:517 —
    on cases with zero padding (pad positions contribute 0 in every encoding), stride 2,
    channel tails inside the packed words (C = 33, 96) and ragged M / OC."""
    for (n, h, w, c, oc, kh, kw, sh, sw, ph, pw) in ((2, 9, 11, 33, 20, 3, 3, 1, 1, 1, 1),
                                                    (1, 12, 10, 96, 100, 3, 3, 2, 2, 1, 1),
                                                    (3, 7, 7, 64, 64, 1, 1, 1, 1, 0, 0)):
        g = inputs.gen(n * 1000 + c + 7 * a_enc + 3 * w_enc + 11 * a_bits + w_bits)
        act = inputs.codes((n, h, w, c), a_bits, g)
        wt = inputs.codes((oc, kh, kw, c), w_bits, g)
        ref = oracle.conv2d_nhwc_enc(act.numpy(), a_bits, a_enc, wt.numpy(), w_bits, w_enc, stride=(sh, sw),
                                     pad=(ph, pw))
        wp = gpu_pack(wt.reshape(oc * kh * kw, c), w_bits)
        w_tc = bs.conv2d_tc_prepare_weights(wp, w_bits, w_enc, oc, kh, kw, c, tc_format=bs.TC_F4)
        got = bs.bitserial_conv2d_nhwc_tc_i8(act.to(DEV), a_bits, w_tc, w_bits, oc, kh, kw, (sh, sw), (ph, pw),
                                             tc_format=bs.TC_F4, a_enc=a_enc, w_enc=w_enc)
        np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"case c={c} a_enc={a_enc} w_enc={w_enc}")


@pytest.mark.parametrize("a_enc,w_enc", ENC_PAIRS)
def test_dense_tc_encodings(a_enc, w_enc):
    """Dense products with every encoding pair, K tails (k = 100, 1000) and a multi-tile
    shape, both entry points (packed / in-call packing)."""
    for (m, n, k, a_bits, w_bits) in ((130, 72, 100, 2, 1), (257, 132, 1000, 3, 2), (64, 256, 4096, 1, 1)):
        a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=a_enc * 100 + w_enc * 10 + a_bits + k)
        ref = oracle.dense_enc(a.numpy(), a_bits, a_enc, w.numpy(), w_bits, w_enc)
        w_tc = bs.dense_tc_prepare_weights(gpu_pack(w, w_bits), w_bits, w_enc, n, k, tc_format=bs.TC_F4)
        got = bs.bitserial_dense_tc_i8(a.to(DEV), a_bits, w_tc, w_bits, n, tc_format=bs.TC_F4, a_enc=a_enc,
                                       w_enc=w_enc)
        np.testing.assert_array_equal(got.cpu().numpy(), ref)
        got2 = bs.bitserial_dense_tc_prepared(gpu_pack(a, a_bits), a_bits, w_tc, w_bits, m, n, k,
                                              tc_format=bs.TC_F4, a_enc=a_enc, w_enc=w_enc)
        assert torch.equal(got, got2)


@pytest.mark.parametrize("w_bits", [1, 2, 3])
def test_i8_signed_weights(w_bits):
    """The I8 format takes signed weights (top plane byte -2^(W-1)); activations unsigned."""
    m, n, k, a_bits = 200, 96, 333, 2
    a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=w_bits + 5)
    ref = oracle.dense_enc(a.numpy(), a_bits, 0, w.numpy(), w_bits, 2)
    w_tc = bs.dense_tc_prepare_weights(gpu_pack(w, w_bits), w_bits, bs.SIGNED, n, k, tc_format=bs.TC_I8)
    got = bs.bitserial_dense_tc_i8(a.to(DEV), a_bits, w_tc, w_bits, n, tc_format=bs.TC_I8, w_enc=bs.SIGNED)
    np.testing.assert_array_equal(got.cpu().numpy(), ref)


# ------------------------------- grouped launch: several convolutions, one persistent kernel
GROUP_CASES = [  # (n, h, w, c, oc, kh, kw, sh, sw, ph, pw): OC <= 64 (N = 64 MMAs), ragged OC
    (2, 9, 11, 33, 20, 3, 3, 1, 1, 1, 1),      # and M tails, stride 2, 1x1, a dense layer
    (1, 12, 10, 96, 100, 3, 3, 2, 2, 1, 1),    # (n = 1, w = 1, 1x1), K from 1 to 36 chunks
    (3, 7, 7, 64, 64, 1, 1, 1, 1, 0, 0),
    (1, 14, 14, 128, 300, 3, 3, 1, 1, 1, 1),
    (1, 130, 1, 1000, 72, 1, 1, 1, 1, 0, 0),
    (2, 5, 5, 7, 4, 3, 3, 1, 1, 2, 2),
]


def _group_run(cases, a_bits, w_bits, fmt, encs, seed):
    items, refs = [], []
    for i, (n, h, w, c, oc, kh, kw, sh, sw, ph, pw) in enumerate(cases):
        a_enc, w_enc = encs[i % len(encs)]
        g = inputs.gen(seed + 31 * i)
        act = inputs.codes((n, h, w, c), a_bits, g)
        wt = inputs.codes((oc, kh, kw, c), w_bits, g)
        refs.append(oracle.conv2d_nhwc_enc(act.numpy(), a_bits, a_enc, wt.numpy(), w_bits, w_enc, stride=(sh, sw),
                                           pad=(ph, pw)))
        w_tc = bs.conv2d_tc_prepare_weights(gpu_pack(wt.reshape(oc * kh * kw, c), w_bits), w_bits, w_enc, oc, kh,
                                            kw, c, tc_format=fmt)
        items.append(dict(act_packed=gpu_pack(act.reshape(-1, c), a_bits), w_tc=w_tc, n=n, h=h, w=w, c=c, oc=oc,
                          kh=kh, kw=kw, stride=(sh, sw), pad=(ph, pw), a_enc=a_enc, w_enc=w_enc))
    return bs.bitserial_conv2d_nhwc_tc_group(items, a_bits, w_bits, tc_format=fmt), refs


@pytest.mark.parametrize("bn", ["", "64", "128"])
@pytest.mark.parametrize("fmt", TC_FORMATS)
@pytest.mark.parametrize("a_bits,w_bits", TC_PRECISIONS)
def test_conv_tc_group_mixed(tuning, bn, fmt, a_bits, w_bits):
    """bs_bitserial_conv2d_nhwc_tc_group on six problems of different geometry (problems
    reordered by K inside; tiles of all problems interleaved across CTAs): every output
    equals the oracle's.  Default tile widths (OC <= 64 members in a BN = 64 group, the
    rest in a BN = 128 group) and every member forced into one BN = 64 or BN = 128
    launch (N = 64 MMAs for the narrow members).  FP4 mixes the encodings per member."""
    if bn:
        tuning(bs.TUNE_TC_TILE_N, int(bn))
    encs = [(bs.A_UNSIGNED, bs.UNIPOLAR), (bs.A_UNSIGNED, bs.BIPOLAR)]
    if fmt == bs.TC_F4:
        encs += [(bs.A_BIPOLAR, bs.BIPOLAR), (bs.A_SIGNED, bs.SIGNED), (bs.A_UNSIGNED, bs.SIGNED)]
    outs, refs = _group_run(GROUP_CASES, a_bits, w_bits, fmt, encs, seed=1000 * fmt + 10 * a_bits + w_bits)
    for i, (o, r) in enumerate(zip(outs, refs)):
        np.testing.assert_array_equal(o.cpu().numpy(), r, err_msg=f"member {i} {GROUP_CASES[i]}")


@pytest.mark.parametrize("split", ["0", "1"])
def test_conv_tc_group_more_than_one_launch(tuning, split):
    """More members than one launch holds (16): split into launches of <= 16, all exact;
    a group of one and an empty group.  split=1: each launch interleaves its long-K and
    short-K members' tiles (BS_TUNE_TC_GROUP_SPLIT)."""
    tuning(bs.TUNE_TC_GROUP_SPLIT, int(split))
    cases = [(1, 4 + i % 5, 5, 16 + 8 * (i % 3), 8 + 12 * (i % 4), 3, 3, 1 + i % 2, 1, 1, 1) for i in range(19)]
    cases += [(2, 6, 6, 512, 72, 3, 3, 1, 1, 1, 1), (3, 5, 7, 8, 100, 1, 1, 1, 1, 0, 0)]  # long / short K
    outs, refs = _group_run(cases, 2, 1, bs.TC_F4, [(bs.A_UNSIGNED, bs.BIPOLAR)], seed=5)
    for i, (o, r) in enumerate(zip(outs, refs)):
        np.testing.assert_array_equal(o.cpu().numpy(), r, err_msg=f"member {i}")
    outs, refs = _group_run(cases[:1], 2, 1, bs.TC_I8, [(bs.A_UNSIGNED, bs.BIPOLAR)], seed=6)
    np.testing.assert_array_equal(outs[0].cpu().numpy(), refs[0])
    assert bs.bitserial_conv2d_nhwc_tc_group([], 2, 1) == []


@pytest.mark.parametrize("fmt", TC_FORMATS)
def test_config4_batch256_tc_group(fmt):
    """BASELINE configs[3] as the bench's grouped step runs it: the ten ResNet-18 layers
    at batch 256, A2W1 bipolar, in ONE grouped launch; each layer equals the single-layer
    launch bit for bit, and the oracle checks images 0 and 255 of every layer."""
    items, acts, wts = [], [], []
    for layer in inputs.BASELINE_LAYERS:
        L = inputs.TABLE1[layer]
        act, wt = inputs.conv_operands(L, 256, 2, 1, inputs.seed_for(4, 2, 1, "bipolar", layer))
        w_tc = bs.conv2d_tc_prepare_weights(gpu_pack(wt.view(L.oc * L.k * L.k, L.ic), 1), 1, bs.BIPOLAR, L.oc, L.k,
                                            L.k, L.ic, tc_format=fmt)
        items.append(dict(act_packed=gpu_pack(act.reshape(-1, L.ic), 2), w_tc=w_tc, n=256, h=L.h, w=L.w, c=L.ic,
                          oc=L.oc, kh=L.k, kw=L.k, stride=L.s, pad=L.pad, w_enc=bs.BIPOLAR))
        acts.append(act)
        wts.append(wt)
    outs = bs.bitserial_conv2d_nhwc_tc_group(items, 2, 1, tc_format=fmt)
    for layer, it, o, act, wt in zip(inputs.BASELINE_LAYERS, items, outs, acts, wts):
        L = inputs.TABLE1[layer]
        single = bs.bitserial_conv2d_nhwc_tc_prepared(it["act_packed"], 2, it["w_tc"], 1, 256, L.h, L.w, L.ic, L.oc,
                                                      L.k, L.k, L.s, L.pad, tc_format=fmt, w_enc=bs.BIPOLAR)
        assert torch.equal(o, single), f"L{layer}"
        o = o.cpu().numpy()
        for img in (0, 255):
            ref = oracle.conv2d_nhwc(act[img:img + 1].numpy(), 2, wt.numpy(), 1, True, stride=(L.s, L.s),
                                     pad=(L.pad, L.pad))
            np.testing.assert_array_equal(o[img:img + 1], ref, err_msg=f"L{layer} image {img}")


def test_bitpack_group_parity():
    """bs_bitpack_group: ragged, unaligned-K, pad-word and multi-launch (> 16 members)
    segments packed in one launch each equal the oracle's packing."""
    shapes = [(3136 * 2, 64), (1001, 96), (513, 4096), (77, 100), (5, 1), (33, 33), (7, 48)] * 3
    for bits in (1, 2, 3, 4, 8):
        g = inputs.gen(bits)
        xs = [inputs.codes(s, bits, g) for s in shapes]
        outs = bs.bitpack_group([x.to(DEV) for x in xs], bits)
        for x, o in zip(xs, outs):
            np.testing.assert_array_equal(o.cpu().numpy().view(np.uint32), oracle.bitpack(x.numpy(), bits))
    assert bs.bitpack_group([], 2) == []


# ------------------------------- fused all-gather epilogue, one GPU
@pytest.mark.parametrize("fmt", TC_FORMATS)
@pytest.mark.parametrize("m,n,k,npeers", [(300, 256, 1000, 2), (128, 64, 64, 1), (257, 132, 4096, 7)])
def test_dense_tc_fused_gather(fmt, m, n, k, npeers):
    """bs_bitserial_dense_tc_prepared_gather as rank 1 of npeers+1 ranks simulated on one
    GPU: the rank's row block of C lands in its own gathered buffer and, from the same
    staged tiles, in every peer's buffer at the same rows; other rows are untouched."""
    world, rank = npeers + 1, 1
    a, w = inputs.dense_operands(m, n, k, 2, 1, seed=m + n + k + npeers)
    ref = oracle.dense(a.numpy(), 2, w.numpy(), 1, True)
    w_tc = bs.dense_tc_prepare_weights(gpu_pack(w, 1), 1, bs.BIPOLAR, n, k, tc_format=fmt)
    fulls = [torch.full((world * m, n), -7, dtype=torch.int32, device=DEV) for _ in range(world)]
    blk = slice(rank * m, (rank + 1) * m)
    peers = [fulls[r][blk] for r in range(world) if r != rank]
    bs.bitserial_dense_tc_gather(gpu_pack(a, 2), 2, w_tc, 1, m, n, k, fulls[rank][blk], peers, tc_format=fmt,
                                 w_enc=bs.BIPOLAR)
    torch.cuda.synchronize()
    for r, f in enumerate(fulls):
        f = f.cpu().numpy()
        np.testing.assert_array_equal(f[blk], ref, err_msg=f"buffer of rank {r}")
        assert (f[:rank * m] == -7).all() and (f[(rank + 1) * m:] == -7).all()


def test_conv_tc_host_group_pipelined():
    """bs_bitserial_conv2d_nhwc_tc_host_group: pinned host activations -> device -> pack ->
    tensor-core conv -> pinned host outputs for several layers on three streams; every
    output equals the oracle (and the call returns only when all are on the host)."""
    cases = [(2, 9, 11, 33, 20, 3, 3, 1, 1), (1, 14, 14, 128, 136, 3, 3, 2, 1), (3, 7, 7, 64, 64, 1, 1, 1, 0)]
    layers, refs = [], []
    for i, (n, h, w, c, oc, kh, kw, st, pd) in enumerate(cases):
        g = inputs.gen(900 + i)
        act = inputs.codes((n, h, w, c), 2, g)
        wt = inputs.codes((oc, kh, kw, c), 1, g)
        refs.append(oracle.conv2d_nhwc(act.numpy(), 2, wt.numpy(), 1, True, stride=(st, st), pad=(pd, pd)))
        w_tc = bs.conv2d_tc_prepare_weights(gpu_pack(wt.reshape(oc * kh * kw, c), 1), 1, bs.BIPOLAR, oc, kh, kw, c)
        oh = bs.conv_out_extent(h, kh, st, pd)
        ow = bs.conv_out_extent(w, kw, st, pd)
        layers.append(dict(act_host=act.contiguous().pin_memory(),
                           out_host=torch.full((n, oh, ow, oc), -9, dtype=torch.int32).pin_memory(),
                           act_dev=torch.empty((n, h, w, c), dtype=torch.uint8, device=DEV),
                           packed_dev=torch.empty(bs.conv2d_workspace_bytes(n, h, w, c, 2) // 4, dtype=torch.int32,
                                                  device=DEV),
                           out_dev=torch.empty((n, oh, ow, oc), dtype=torch.int32, device=DEV), w_tc=w_tc, oc=oc,
                           kh=kh, kw=kw, stride=st, pad=pd, w_enc=bs.BIPOLAR))
    for _ in range(2):  # repeated calls reuse the buffers
        outs = bs.bitserial_conv2d_nhwc_tc_host_group(layers, 2, 1)
        for o, r in zip(outs, refs):
            np.testing.assert_array_equal(o.numpy(), r)


@pytest.mark.parametrize("fmt", TC_FORMATS)
@pytest.mark.parametrize("size", [4096, 8192, 16384])
@pytest.mark.parametrize("a_bits,w_bits,bipolar", [(1, 1, False), (2, 1, True), (4, 2, True)])
def test_config5_gemm_tc_sampled_rows(fmt, size, a_bits, w_bits, bipolar):
    """BASELINE configs[4] on the tensor-core path in the bench's launch configuration
    (bs_bitserial_dense_tc_i8: activation pack + one persistent launch over the whole
    M = N = K product); the oracle checks rows at both ends and the middle, every column."""
    e = "bipolar" if bipolar else "unipolar"
    a, w = inputs.dense_operands(size, size, size, a_bits, w_bits, inputs.seed_for(5, a_bits, w_bits, e))
    w_tc = bs.dense_tc_prepare_weights(gpu_pack(w, w_bits), w_bits, enc(bipolar), size, size, tc_format=fmt)
    got = bs.bitserial_dense_tc_i8(a.to(DEV), a_bits, w_tc, w_bits, size, tc_format=fmt, w_enc=enc(bipolar))
    rows = [0, 127, 128, size // 2 + 3, size - 1]
    ref = oracle.dense(a[rows].numpy(), a_bits, w.numpy(), w_bits, bipolar)
    np.testing.assert_array_equal(got[rows].cpu().numpy(), ref)
    del got
    torch.cuda.empty_cache()


@pytest.mark.parametrize("fmt", TC_FORMATS)
def test_tc_group_writes_stay_in_bounds(fmt):
    """Every grouped-launch output lives inside one flat buffer between sentinel guard
    bands (ragged M / OC, OC % 4 != 0 scalar epilogue, OC <= 64 and wide members): the
    outputs equal the oracle and no byte outside them changes."""
    cases = [(1, 9, 11, 33, 20, 3, 3, 1, 1), (2, 5, 7, 64, 130, 3, 3, 2, 1), (1, 6, 6, 96, 18, 1, 1, 1, 0),
             (3, 7, 5, 40, 64, 3, 3, 1, 1)]
    guard = 4096
    sizes = []
    for (n, h, w, c, oc, kh, kw, st, pd) in cases:
        oh, ow = bs.conv_out_extent(h, kh, st, pd), bs.conv_out_extent(w, kw, st, pd)
        sizes.append((n, oh, ow, oc))
    total = guard + sum(int(np.prod(s_)) + guard for s_ in sizes)
    flat = torch.full((total,), 0x5A5A5A5A, dtype=torch.int32, device=DEV)
    items, refs, spans, off = [], [], [], guard
    for i, ((n, h, w, c, oc, kh, kw, st, pd), shp) in enumerate(zip(cases, sizes)):
        g = inputs.gen(700 + i)
        act = inputs.codes((n, h, w, c), 2, g)
        wt = inputs.codes((oc, kh, kw, c), 1, g)
        refs.append(oracle.conv2d_nhwc(act.numpy(), 2, wt.numpy(), 1, True, stride=(st, st), pad=(pd, pd)))
        cnt = int(np.prod(shp))
        out = flat[off:off + cnt].view(shp)
        spans.append((off, cnt))
        off += cnt + guard
        w_tc = bs.conv2d_tc_prepare_weights(gpu_pack(wt.reshape(oc * kh * kw, c), 1), 1, bs.BIPOLAR, oc, kh, kw, c,
                                            tc_format=fmt)
        items.append(dict(act_packed=gpu_pack(act.reshape(-1, c), 2), w_tc=w_tc, out=out, n=n, h=h, w=w, c=c, oc=oc,
                          kh=kh, kw=kw, stride=st, pad=pd, w_enc=bs.BIPOLAR))
    bs.bitserial_conv2d_nhwc_tc_group(items, 2, 1, tc_format=fmt)
    host = flat.cpu().numpy()
    mask = np.ones(total, dtype=bool)
    for (o, cnt), shp, r in zip(spans, sizes, refs):
        np.testing.assert_array_equal(host[o:o + cnt].reshape(shp), r)
        mask[o:o + cnt] = False
    assert (host[mask] == 0x5A5A5A5A).all()


@pytest.mark.parametrize("fmt", TC_FORMATS)
@pytest.mark.parametrize("bn", ["64", "128"])
@pytest.mark.parametrize("a_bits,w_bits", [(2, 1), (4, 3), (1, 4)])
def test_tc_single_launch_writes_stay_in_bounds(tuning, fmt, bn, a_bits, w_bits):
    """A single tensor-core launch (ragged M and OC, each tile width) writes exactly its
    output: sentinel guard bands before and after stay intact."""
    tuning(bs.TUNE_TC_TILE_N, int(bn))
    n, h, w, c, oc = 2, 11, 9, 72, 100
    g = inputs.gen(31 * a_bits + w_bits + int(bn))
    act = inputs.codes((n, h, w, c), a_bits, g)
    wt = inputs.codes((oc, 3, 3, c), w_bits, g)
    ref = oracle.conv2d_nhwc(act.numpy(), a_bits, wt.numpy(), w_bits, True, stride=(1, 1), pad=(1, 1))
    guard, cnt = 4096, ref.size
    flat = torch.full((2 * guard + cnt,), 0x3C3C3C3C, dtype=torch.int32, device=DEV)
    out = flat[guard:guard + cnt].view(ref.shape)
    w_tc = bs.conv2d_tc_prepare_weights(gpu_pack(wt.reshape(oc * 9, c), w_bits), w_bits, bs.BIPOLAR, oc, 3, 3, c,
                                        tc_format=fmt)
    bs.bitserial_conv2d_nhwc_tc_prepared(gpu_pack(act.reshape(-1, c), a_bits), a_bits, w_tc, w_bits, n, h, w, c, oc,
                                         3, 3, 1, 1, out=out, tc_format=fmt, w_enc=bs.BIPOLAR)
    host = flat.cpu().numpy()
    np.testing.assert_array_equal(host[guard:guard + cnt].reshape(ref.shape), ref)
    assert (host[:guard] == 0x3C3C3C3C).all() and (host[guard + cnt:] == 0x3C3C3C3C).all()


# ------------------------------------------------- one-launch small-problem path (N6)
SMALL_CASES = CONV_CASES + [(1, 1, 300, 100, 70, 1, 1, 1, 1, 0, 0),   # dense 300 x 70, k = 100
                            (1, 1, 17, 4096, 130, 1, 1, 1, 1, 0, 0)]  # dense 17 x 130, k = 4096


def _small_run(cases, a_bits, w_bits, encs, seed):
    items, refs = [], []
    for i, (n, h, w, c, oc, kh, kw, sh, sw, ph, pw) in enumerate(cases):
        g = inputs.gen(seed * 1000 + i)
        act = inputs.codes((n, h, w, c), a_bits, g)
        wt = inputs.codes((oc, kh, kw, c), w_bits, g)
        we = encs[i % len(encs)]
        refs.append(oracle.conv2d_nhwc(act.numpy(), a_bits, wt.numpy(), w_bits, we == bs.BIPOLAR, stride=(sh, sw),
                                       pad=(ph, pw)))
        items.append(dict(act=act.to(DEV), w_packed=gpu_pack(wt.view(oc * kh * kw, c), w_bits), w_enc=we, oc=oc,
                          kh=kh, kw=kw, stride=(sh, sw), pad=(ph, pw)))
    return bs.bitserial_conv2d_nhwc_i8_group(items, a_bits, w_bits), refs


@pytest.mark.parametrize("ks", [0, 1, 2, 4, 8])
@pytest.mark.parametrize("a_bits,w_bits", [(1, 1), (2, 1), (2, 2), (3, 1), (4, 2), (1, 2)])
def test_small_group_ragged(tuning, ks, a_bits, w_bits):
    """bs_bitserial_conv2d_nhwc_i8_group (fused packing, AND+POPC, K slices of a tile summed
    through distributed shared memory) on the ragged conv cases and two dense layers, every
    K split (0 = automatic), unipolar and bipolar members in one launch: exact."""
    if ks:
        tuning(bs.TUNE_SMALL_KSPLIT, ks)
    outs, refs = _small_run(SMALL_CASES, a_bits, w_bits, [bs.UNIPOLAR, bs.BIPOLAR], seed=10 * a_bits + w_bits + ks)
    for i, (o, r) in enumerate(zip(outs, refs)):
        np.testing.assert_array_equal(o.cpu().numpy(), r, err_msg=f"member {i} {SMALL_CASES[i]}")


@pytest.mark.parametrize("a_bits,w_bits", [(1, 1), (2, 1), (2, 2)])
@pytest.mark.parametrize("bipolar", [False, True])
def test_small_group_resnet_batch1(a_bits, w_bits, bipolar):
    """BASELINE configs[2]: the ten ResNet-18 layers at batch 1 in ONE launch of the small
    path (the bench's resnet1 step), every output vs the oracle."""
    cases = [(1, L.h, L.w, L.ic, L.oc, L.k, L.k, L.s, L.s, L.pad, L.pad)
             for L in (inputs.TABLE1[li] for li in inputs.BASELINE_LAYERS)]
    enc_ = bs.BIPOLAR if bipolar else bs.UNIPOLAR
    outs, refs = _small_run(cases, a_bits, w_bits, [enc_], seed=77 + a_bits * 10 + w_bits)
    for li, o, r in zip(inputs.BASELINE_LAYERS, outs, refs):
        np.testing.assert_array_equal(o.cpu().numpy(), r, err_msg=f"layer {li}")


def test_small_group_validation():
    """Unsupported precisions / signed weights are refused before launch; more than 16
    members run as consecutive launches; an empty group is a no-op."""
    g = inputs.gen(3)
    act = inputs.codes((1, 5, 5, 8), 2, g).to(DEV)
    wt = gpu_pack(inputs.codes((4, 8), 3, g), 3)
    with pytest.raises(bs.BitserialError, match="UNSUPPORTED"):
        bs.bitserial_conv2d_nhwc_i8_group([dict(act=act, w_packed=wt, oc=4, kh=1, kw=1)], 2, 3)
    wt1 = gpu_pack(inputs.codes((4, 8), 1, g), 1)
    with pytest.raises(bs.BitserialError, match="UNSUPPORTED|INVALID_ARG"):
        bs.bitserial_conv2d_nhwc_i8_group([dict(act=act, w_packed=wt1, w_enc=bs.SIGNED, oc=4, kh=1, kw=1)], 2, 1)
    assert bs.bitserial_conv2d_nhwc_i8_group([], 2, 1) == []
    cases = [(1, 3 + i % 4, 4 + i % 3, 8 + 8 * (i % 5), 5 + 3 * i, 3, 3, 1 + i % 2, 1, 1, 1) for i in range(19)]
    outs, refs = _small_run(cases, 2, 1, [bs.BIPOLAR, bs.UNIPOLAR], seed=4)
    for i, (o, r) in enumerate(zip(outs, refs)):
        np.testing.assert_array_equal(o.cpu().numpy(), r, err_msg=f"member {i}")


# ------------------------------- the three-call boundary on the tensor cores (packed weights)
THREE_CALL_CONV = [(2, 13, 11, 96, 40, 3, 3, 1, 1, 1, 1), (3, 10, 10, 64, 300, 3, 3, 2, 2, 1, 1),
                   (1, 9, 7, 5, 3, 3, 3, 1, 1, 1, 1), (2, 5, 9, 17, 6, 2, 3, 3, 1, 2, 0),
                   (2, 7, 7, 512, 64, 3, 3, 1, 1, 1, 1), (4, 14, 14, 256, 130, 3, 3, 1, 1, 1, 1),
                   (2, 8, 8, 64, 128, 1, 1, 2, 2, 0, 0)]


@pytest.mark.parametrize("case", THREE_CALL_CONV)
@pytest.mark.parametrize("a_bits,w_bits", [(1, 1), (2, 1), (2, 2), (4, 2), (3, 3), (4, 4)])
@pytest.mark.parametrize("bipolar", [False, True])
def test_three_call_conv_tc(case, a_bits, w_bits, bipolar):
    """bs_bitpack + bs_bitserial_conv2d_nhwc (BS_ALGO_AUTO -> the tensor-core kernel on the
    PACKED weight planes, expanded in shared memory by the producer warps) and BS_ALGO_TC
    explicitly: exact on ragged geometries, every precision A, W <= 4, both encodings."""
    n, h, w, c, oc, kh, kw, sh, sw, ph, pw = case
    g = inputs.gen(sum(case) * 13 + a_bits * 7 + w_bits + (1000 if bipolar else 0))
    act = inputs.codes((n, h, w, c), a_bits, g)
    wt = inputs.codes((oc, kh, kw, c), w_bits, g)
    ref = oracle.conv2d_nhwc(act.numpy(), a_bits, wt.numpy(), w_bits, bipolar, stride=(sh, sw), pad=(ph, pw))
    ap = gpu_pack(act.view(-1, c), a_bits)
    wp = gpu_pack(wt.view(oc * kh * kw, c), w_bits)
    for algo in (bs.ALGO_AUTO, bs.ALGO_TC):
        got = bs.bitserial_conv2d_nhwc(ap, a_bits, wp, w_bits, enc(bipolar), n, h, w, c, oc, kh, kw, (sh, sw),
                                       (ph, pw), algo=algo)
        np.testing.assert_array_equal(got.cpu().numpy(), ref, err_msg=f"algo {algo}")


@pytest.mark.parametrize("slots", [0, 2, 3])
@pytest.mark.parametrize("bn", [0, 64, 128])
def test_three_call_conv_tc_weight_slots(tuning, slots, bn):
    """Packed-weight tensor-core launches with the weight chunks resident (loaded once per N
    block and CTA) and streamed through 2 or 3 slots (every chunk re-expanded by the producer
    team that handles it), both tile widths, 3 N blocks, 18 K chunks."""
    if slots:
        tuning(bs.TUNE_TC_B_SLOTS, slots)
    if bn:
        tuning(bs.TUNE_TC_TILE_N, bn)
    n, h, w, c, oc = 2, 9, 9, 512, 300
    for bipolar in (False, True):
        g = inputs.gen(slots * 10 + bn + bipolar)
        act = inputs.codes((n, h, w, c), 2, g)
        wt = inputs.codes((oc, 3, 3, c), 2, g)
        ref = oracle.conv2d_nhwc(act.numpy(), 2, wt.numpy(), 2, bipolar, stride=(1, 1), pad=(1, 1))
        got = bs.bitserial_conv2d_nhwc(gpu_pack(act.view(-1, c), 2), 2, gpu_pack(wt.view(oc * 9, c), 2), 2,
                                       enc(bipolar), n, h, w, c, oc, 3, 3, 1, 1, algo=bs.ALGO_TC)
        np.testing.assert_array_equal(got.cpu().numpy(), ref)


@pytest.mark.parametrize("m,n,k", [(9, 7, 33), (129, 65, 250), (300, 200, 576), (257, 130, 1000), (64, 256, 4096)])
@pytest.mark.parametrize("a_bits,w_bits", [(1, 1), (2, 1), (2, 2), (4, 1)])
def test_three_call_dense_tc(m, n, k, a_bits, w_bits):
    """bs_bitserial_dense (AUTO: the tensor-core kernel on packed weights for m > 8)."""
    for bipolar in (False, True):
        a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=m + n + k + 10 * a_bits + w_bits + bipolar)
        ref = oracle.dense(a.numpy(), a_bits, w.numpy(), w_bits, bipolar)
        for algo in (bs.ALGO_AUTO, bs.ALGO_TC):
            got = bs.bitserial_dense(gpu_pack(a, a_bits), a_bits, gpu_pack(w, w_bits), w_bits, enc(bipolar), m, n, k,
                                     algo=algo)
            np.testing.assert_array_equal(got.cpu().numpy(), ref)


def test_three_call_tc_refusals():
    """BS_ALGO_TC outside its domain is refused before launch: W = 6, and the FP4 bound."""
    a = gpu_pack(torch.ones((4, 64), dtype=torch.uint8), 2)
    w6 = gpu_pack(torch.ones((4, 64), dtype=torch.uint8), 6)
    with pytest.raises(bs.BitserialError, match="UNSUPPORTED"):
        bs.bitserial_dense(a, 2, w6, 6, bs.UNIPOLAR, 4, 4, 64, algo=bs.ALGO_TC)
    k = 18_642
    a4 = gpu_pack(torch.full((2, k), 15, dtype=torch.uint8), 4)
    w4 = gpu_pack(torch.full((3, k), 15, dtype=torch.uint8), 4)
    with pytest.raises(bs.BitserialError, match="UNSUPPORTED"):
        bs.bitserial_dense(a4, 4, w4, 4, bs.UNIPOLAR, 2, 3, k, algo=bs.ALGO_TC)
    # AUTO past the bound falls back to the integer pipes, still exact
    got = bs.bitserial_dense(a4, 4, w4, 4, bs.UNIPOLAR, 2, 3, k)
    assert int(got[0, 0]) == k * 225


def test_three_call_headline_config():
    """BASELINE configs[3] (ten ResNet-18 layers, batch 256, A2W1 bipolar) through the
    north_star's three calls only — bs_bitpack of the activations and bs_bitserial_conv2d_nhwc
    on packed weights (AUTO: tensor cores) — every layer checked against the oracle on
    sampled images; the step time is compared with the grouped prepared-weight step."""
    import time
    runs = []
    for li in inputs.BASELINE_LAYERS:
        L = inputs.TABLE1[li]
        act, wt = inputs.conv_operands(L, 256, 2, 1, inputs.seed_for(4, 2, 1, "bipolar", li))
        wp = gpu_pack(wt.view(L.oc * L.k * L.k, L.ic), 1)
        runs.append((L, act, wt, act.to(DEV), wp))

    def step(outs=None):
        res = []
        for L, _, _, act_d, wp in runs:
            ap = bs.bitpack(act_d.view(-1, L.ic), 2)
            res.append(bs.bitserial_conv2d_nhwc(ap, 2, wp, 1, bs.BIPOLAR, 256, L.h, L.w, L.ic, L.oc, L.k, L.k, L.s,
                                                L.pad))
        return res
    outs = step()
    torch.cuda.synchronize()
    for (L, act, wt, _, _), o in zip(runs, outs):
        for img in (0, 131, 255):
            ref = oracle.conv2d_nhwc(act[img:img + 1].numpy(), 2, wt.numpy(), 1, True, stride=(L.s, L.s),
                                     pad=(L.pad, L.pad))
            np.testing.assert_array_equal(o[img:img + 1].cpu().numpy(), ref, err_msg=f"layer {L}")
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        step()
    e1.record()
    torch.cuda.synchronize()
    print(f"three-call step: {e0.elapsed_time(e1) / 5:.3f} ms")


def test_dense_tc_multicast_epilogue_single_device():
    """The NVLS form of the fused all-gather (bs_bitserial_dense_tc_prepared_multicast): the
    epilogue stores every row segment with multimem.st to a multicast address.  On one GPU a
    multicast object bound to that device alone stands in for the NVSwitch group: the C
    read back through the unicast mapping equals the oracle (multi-GPU replication is
    unverified here)."""
    from paper_1810_11066_b200.dist import SingleDeviceMulticast
    m, n, k = 300, 200, 576
    try:
        mc = SingleDeviceMulticast(m * n * 4)
    except Exception as e:  # noqa: BLE001
        pytest.skip(f"multicast not available on this device/driver: {e}")
    try:
        for a_bits, w_bits, bipolar in ((2, 1, True), (4, 2, False)):
            a, w = inputs.dense_operands(m, n, k, a_bits, w_bits, seed=a_bits * 10 + w_bits)
            ref = oracle.dense(a.numpy(), a_bits, w.numpy(), w_bits, bipolar)
            w_tc = bs.dense_tc_prepare_weights(gpu_pack(w, w_bits), w_bits, enc(bipolar), n, k)
            bs.bitserial_dense_tc_multicast(gpu_pack(a, a_bits), a_bits, w_tc, w_bits, m, n, k, mc.multicast_ptr(),
                                            w_enc=enc(bipolar))
            got = mc.read(m * n * 4).view(torch.int32).view(m, n).numpy()
            np.testing.assert_array_equal(got, ref)
    finally:
        mc.close()
