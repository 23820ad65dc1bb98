"""CPU oracle for the bitserial hot path (arXiv 1810.11066) — TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product package
``paper_1810_11066_b200`` never imports it and shares no code with it.

The arithmetic lives in ``oracle/oracle.c`` (plain C, OpenMP over the outermost
output loop).  This module only builds that library with gcc and marshals numpy
arrays into it.  Every function states the passage it follows; the pins that tie
it to the paper are in ``tests/test_oracle_pins.py``.

Parity status: every function below is pinned (no "parity unpinned" entries); see
DESIGN.md §3 for the readings of the paper they rely on.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c into oracle/liboracle.so with gcc (-O3 -march=native -fopenmp)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        tmp = _LIB_PATH + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O3", "-march=native", "-fopenmp", "-fPIC", "-shared",
                               "-Wall", "-Wextra", "-o", tmp, _SRC])
        os.replace(tmp, _LIB_PATH)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        P, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        lib.oracle_weight_value.argtypes = [I, I, I]
        lib.oracle_weight_value.restype = L
        lib.oracle_dense.argtypes = [P, I, P, I, I, P, L, L, L]
        lib.oracle_dense.restype = I
        lib.oracle_conv2d_nhwc.argtypes = [P, I, P, I, I, P] + [I] * 11
        lib.oracle_conv2d_nhwc.restype = I
        lib.oracle_conv_out_extent.argtypes = [L, L, L, L]
        lib.oracle_conv_out_extent.restype = L
        lib.oracle_packed_row_words.argtypes = [L]
        lib.oracle_packed_row_words.restype = L
        lib.oracle_bitpack.argtypes = [P, P, L, L, I]
        lib.oracle_bitpack.restype = I
        lib.oracle_num_threads.restype = I
        lib.oracle_code_value.argtypes = [I, I, I]
        lib.oracle_code_value.restype = L
        lib.oracle_dense_enc.argtypes = [P, I, I, P, I, I, P, L, L, L]
        lib.oracle_dense_enc.restype = I
        lib.oracle_conv2d_nhwc_enc.argtypes = [P, I, I, P, I, I, P] + [I] * 11
        lib.oracle_conv2d_nhwc_enc.restype = I
        lib.oracle_e2m1_twice.argtypes = [I]
        lib.oracle_e2m1_twice.restype = I
        lib.oracle_digit_value.argtypes = [I, I, I, I]
        lib.oracle_digit_value.restype = I
        lib.oracle_digitpack.argtypes = [P, P, L, L, I, I]
        lib.oracle_digitpack.restype = I
        _lib = lib
    return _lib


def _u8(x) -> np.ndarray:
    x = np.asarray(x)
    if x.dtype != np.uint8:
        if x.size and (x.min() < 0 or x.max() > 255):
            raise ValueError("codes must lie in [0, 255]")
        x = x.astype(np.uint8)
    return np.ascontiguousarray(x)


def _ptr(x: np.ndarray):
    return x.ctypes.data_as(ctypes.c_void_p)


def num_threads() -> int:
    """OpenMP threads the oracle runs on (OMP_NUM_THREADS, else all host cores)."""
    return int(_load().oracle_num_threads())


def weight_value(code: int, bits: int, bipolar: bool) -> int:
    """Value of one weight code: unipolar = code; bipolar = sum_j 2^j (2 b_j - 1)
    (PAPER.md:503 bipolar +/-1 digits; readings R1-R3)."""
    return int(_load().oracle_weight_value(int(code), int(bits), int(bool(bipolar))))


def dense(a, a_bits: int, w, w_bits: int, bipolar: bool) -> np.ndarray:
    """out[m][n] = sum_k a[m][k] * value(w[n][k]).

    a: [M][K] unsigned activation codes; w: [N][K] weight codes; returns int32 [M][N]."""
    a, w = _u8(a), _u8(w)
    if a.ndim != 2 or w.ndim != 2 or a.shape[1] != w.shape[1]:
        raise ValueError("dense: a [M][K], w [N][K] with equal K")
    m, k = a.shape
    n = w.shape[0]
    out = np.empty((m, n), dtype=np.int32)
    rc = _load().oracle_dense(_ptr(a), a_bits, _ptr(w), w_bits, int(bool(bipolar)), _ptr(out), m, n, k)
    if rc != 0:
        raise ValueError("oracle_dense rejected its arguments")
    return out


def conv_out_extent(size: int, k: int, stride: int, pad: int) -> int:
    """floor((size + 2 pad - k) / stride) + 1, or 0 if the window does not fit."""
    return int(_load().oracle_conv_out_extent(size, k, stride, pad))


def conv2d_nhwc(act, a_bits: int, wt, w_bits: int, bipolar: bool,
                stride=(1, 1), pad=(0, 0)) -> np.ndarray:
    """NHWC cross-correlation with zero padding, OHWI weights (Table 1
    PAPER.md:733-746).  act: [N][H][W][C] codes; wt: [OC][KH][KW][C] codes;
    returns int32 [N][OH][OW][OC]."""
    act, wt = _u8(act), _u8(wt)
    if act.ndim != 4 or wt.ndim != 4 or act.shape[3] != wt.shape[3]:
        raise ValueError("conv2d_nhwc: act [N][H][W][C], wt [OC][KH][KW][C]")
    n, h, w, c = act.shape
    oc, kh, kw, _ = wt.shape
    sh, sw = stride
    ph, pw = pad
    oh, ow = conv_out_extent(h, kh, sh, ph), conv_out_extent(w, kw, sw, pw)
    if oh <= 0 or ow <= 0:
        raise ValueError("conv2d_nhwc: empty output")
    out = np.empty((n, oh, ow, oc), dtype=np.int32)
    rc = _load().oracle_conv2d_nhwc(_ptr(act), a_bits, _ptr(wt), w_bits, int(bool(bipolar)), _ptr(out),
                                    n, h, w, c, oc, kh, kw, sh, sw, ph, pw)
    if rc != 0:
        raise ValueError("oracle_conv2d_nhwc rejected its arguments")
    return out


UNSIGNED, BIPOLAR, SIGNED = 0, 1, 2  # operand encodings of the *_enc functions


def code_value(code: int, bits: int, enc: int) -> int:
    """Value of one code: 0 unsigned = code; 1 bipolar = sum_j 2^j (2 b_j - 1)
    (PAPER.md:503); 2 signed two's complement, top plane -2^(bits-1)."""
    return int(_load().oracle_code_value(int(code), int(bits), int(enc)))


def dense_enc(a, a_bits: int, a_enc: int, w, w_bits: int, w_enc: int) -> np.ndarray:
    """out[m][n] = sum_k value(a[m][k]) * value(w[n][k]) with an encoding per operand
    (both-bipolar XNOR form PAPER.md:503, signed data PAPER.md:517)."""
    a, w = _u8(a), _u8(w)
    if a.ndim != 2 or w.ndim != 2 or a.shape[1] != w.shape[1]:
        raise ValueError("dense_enc: a [M][K], w [N][K] with equal K")
    m, k = a.shape
    n = w.shape[0]
    out = np.empty((m, n), dtype=np.int32)
    if _load().oracle_dense_enc(_ptr(a), a_bits, a_enc, _ptr(w), w_bits, w_enc, _ptr(out), m, n, k) != 0:
        raise ValueError("oracle_dense_enc rejected its arguments")
    return out


def conv2d_nhwc_enc(act, a_bits: int, a_enc: int, wt, w_bits: int, w_enc: int,
                    stride=(1, 1), pad=(0, 0)) -> np.ndarray:
    """conv2d_nhwc with an encoding per operand; padded positions contribute 0."""
    act, wt = _u8(act), _u8(wt)
    if act.ndim != 4 or wt.ndim != 4 or act.shape[3] != wt.shape[3]:
        raise ValueError("conv2d_nhwc_enc: act [N][H][W][C], wt [OC][KH][KW][C]")
    n, h, w, c = act.shape
    oc, kh, kw, _ = wt.shape
    sh, sw = stride
    ph, pw = pad
    oh, ow = conv_out_extent(h, kh, sh, ph), conv_out_extent(w, kw, sw, pw)
    if oh <= 0 or ow <= 0:
        raise ValueError("conv2d_nhwc_enc: empty output")
    out = np.empty((n, oh, ow, oc), dtype=np.int32)
    rc = _load().oracle_conv2d_nhwc_enc(_ptr(act), a_bits, a_enc, _ptr(wt), w_bits, w_enc, _ptr(out),
                                        n, h, w, c, oc, kh, kw, sh, sw, ph, pw)
    if rc != 0:
        raise ValueError("oracle_conv2d_nhwc_enc rejected its arguments")
    return out


def packed_row_words(k: int) -> int:
    """Words per packed row: ceil(k/32) rounded up to even (reading R7)."""
    return int(_load().oracle_packed_row_words(k))


def bitpack(x, bits: int) -> np.ndarray:
    """Bit-plane packing, layout BMK': returns uint32
    [bits][rows][Kw_pad]; bit t of word j of plane b = bit b of x[r][32 j + t]."""
    x = _u8(x)
    if x.ndim != 2:
        raise ValueError("bitpack: x [rows][K]")
    rows, k = x.shape
    out = np.empty((bits, rows, packed_row_words(k)), dtype=np.uint32)
    if _load().oracle_bitpack(_ptr(x), _ptr(out), rows, k, bits) != 0:
        raise ValueError("oracle_bitpack rejected its arguments")
    return out


def e2m1_twice(nib: int) -> int:
    """2 x the value of a 4-bit E2M1 field (sign bit 3, exponent bits 2..1, mantissa bit 0)."""
    return int(_load().oracle_e2m1_twice(int(nib)))


def digit_value(code: int, bits: int, enc: int, d: int) -> int:
    """Radix-4 digit d of a code (planes 2d, 2d+1; R21/R24) in its encoding."""
    return int(_load().oracle_digit_value(int(code), int(bits), int(enc), int(d)))


def digit_row_bytes(k: int) -> int:
    """Bytes per digit-packed row: 16 x packed_row_words(k) (4 bits per element)."""
    return 16 * packed_row_words(k)


def digitpack(x, bits: int, enc: int = UNSIGNED) -> np.ndarray:
    """Digit packing (the C ABI's digit-packed layout, R24): uint8
    [ceil(bits/2)][rows][digit_row_bytes(k)], element t of a row in nibble t % 2 of byte
    t // 2, holding the E2M1 code of 0.5 x its digit value; zero past k."""
    x = _u8(x)
    if x.ndim != 2:
        raise ValueError("digitpack: x [rows][K]")
    rows, k = x.shape
    out = np.empty(((bits + 1) // 2, rows, digit_row_bytes(k)), dtype=np.uint8)
    if _load().oracle_digitpack(_ptr(x), _ptr(out), rows, k, bits, enc) != 0:
        raise ValueError("oracle_digitpack rejected its arguments")
    return out


# ---------------------------------------------------------------- window layout (R26)
def win_geometry(n: int, h: int, w: int, c: int, kh: int, kw: int, stride: int, pad_h: int, pad_w: int) -> dict:
    """Geometry of the window layout (reading R26), written out from its definition.

    The conv's zero-padded input (PAPER.md:573 NHWC conv; padding = value 0, reading R20) is
    split into the stride x stride phases (py, px) its taps read: phase pixel (gy, gx) is padded
    pixel (gy*s + py, gx*s + px).  Output (oy, ox) with tap (ky, kx) reads phase
    (ky % s, kx % s) at (oy + ky // s, ox + kx // s), so on a phase grid of hg x wg pixels per
    image (flattened q = (img*hg + gy)*wg + gx) it reads q_out + (ky // s)*wg + kx // s.
    """
    s = stride
    oh = conv_out_extent(h, kh, s, pad_h)
    ow = conv_out_extent(w, kw, s, pad_w)
    hg = oh + (kh - 1) // s
    wg = ow + (kw - 1) // s
    phases = sorted({(ky % s) * s + (kx % s) for ky in range(kh) for kx in range(kw)})
    maxoff = ((kh - 1) // s) * wg + (kw - 1) // s
    lwin = (128 + maxoff + 8 + 7) // 8 * 8       # rows a 128-row tile reads per window (from an 8-row boundary)
    gpix = n * hg * wg
    pstride = (gpix + lwin + 7) // 8 * 8         # zero tail: the last tile's window stays inside
    cw = packed_row_words(c)
    return dict(s=s, oh=oh, ow=ow, hg=hg, wg=wg, phases=phases, nph=len(phases), maxoff=maxoff, lwin=lwin,
                gpix=gpix, pstride=pstride, cw=cw, pairs=cw // 2)


def _swap_halves(rows32: np.ndarray, r: np.ndarray) -> np.ndarray:
    """32-byte rows with their two 16-byte halves exchanged where bit 2 of the row index r is
    set (the 32-byte shared-memory swizzle the rows are stored in, R26)."""
    out = rows32.copy()
    sw = ((r >> 2) & 1).astype(bool)
    out[..., sw, :16] = rows32[..., sw, 16:]
    out[..., sw, 16:] = rows32[..., sw, :16]
    return out


def digitpack_win(x, bits: int, enc: int, kh: int, kw: int, stride: int, pad_h: int, pad_w: int) -> np.ndarray:
    """Window layout of NHWC activation codes x [n][h][w][c] (R26): uint8
    [D][nph][pairs][pstride][32], D = ceil(bits/2), pairs = cw / 2.  Row (d, phase slot, pair p,
    q) holds the 16 digit-packed bytes (oracle.digitpack, R24) of channels [64p, 64p+32) and of
    [64p+32, 64p+64) of the input pixel that phase-grid position q maps to — in that order, or
    exchanged when bit 2 of q is set — or zeros where q is padding, lies past the image, or is
    in the tail (q >= n*hg*wg)."""
    x = _u8(x)
    if x.ndim != 4:
        raise ValueError("digitpack_win: x [n][h][w][c]")
    n, h, w, c = x.shape
    g = win_geometry(n, h, w, c, kh, kw, stride, pad_h, pad_w)
    s, hg, wg, cw, ps = g["s"], g["hg"], g["wg"], g["cw"], g["pstride"]
    dig = digitpack(x.reshape(n * h * w, c), bits, enc)          # [D][pixels][16*cw]
    D = dig.shape[0]
    plain = np.zeros((D, g["nph"], cw // 2, ps, 32), dtype=np.uint8)
    q = np.arange(g["gpix"])
    img, rem = q // (hg * wg), q % (hg * wg)
    gy, gx = rem // wg, rem % wg
    for f, phase in enumerate(g["phases"]):
        py, px = phase // s, phase % s
        y = gy * s + py - pad_h
        xx = gx * s + px - pad_w
        ok = (y >= 0) & (y < h) & (xx >= 0) & (xx < w)
        pix = (img[ok] * h + y[ok]) * w + xx[ok]
        for p in range(cw // 2):
            plain[:, f, p, q[ok], :] = dig[:, pix, 32 * p:32 * p + 32]
    return _swap_halves(plain, np.arange(ps))


def conv2d_tcw_weights(wt, w_bits: int, w_enc: int) -> np.ndarray:
    """Window-path weight digits of OHWI weight codes wt [oc][kh][kw][c] (R26):
    uint8 [nblk][pairs][Dw][kh*kw][BN][32], BN = 64 if oc <= 64 else 128,
    nblk = ceil(oc / BN), pairs = cw / 2; row (nb, p, e, tap, r) holds the digit bytes
    (oracle.digitpack) of channels [64p, 64p+64) of filter nb*BN + r at that tap, its two
    16-byte halves exchanged when bit 2 of r is set (zeros for filters >= oc)."""
    wt = _u8(wt)
    oc, kh, kw, c = wt.shape
    bn = 64 if oc <= 64 else 128
    nblk = (oc + bn - 1) // bn
    cw = packed_row_words(c)
    dig = digitpack(wt.reshape(oc * kh * kw, c), w_bits, w_enc)   # [Dw][oc*taps][16*cw]
    D = dig.shape[0]
    taps = kh * kw
    full = np.zeros((D, nblk * bn, taps, cw // 2, 32), dtype=np.uint8)
    full[:, :oc] = dig.reshape(D, oc, taps, cw // 2, 32)
    # [e][nb][r][tap][p][32] -> [nb][p][e][tap][r][32]
    t = np.ascontiguousarray(full.reshape(D, nblk, bn, taps, cw // 2, 32).transpose(1, 4, 0, 3, 2, 5))
    return _swap_halves(t, np.arange(bn))
