"""Python binding of the B200 bitserial C ABI (include/bitserial.h).

Argument marshalling only: every function checks tensor placement/dtype/shape,
allocates outputs with torch (device memory is PyTorch's job), and calls the
same-named ``bs_*`` entry point of ``libbitserial.so`` on the current CUDA stream.
All arithmetic of the hot path runs in the library's sm_100a kernels; there is no
CPU fallback — if the library is missing or the device is not CUDA, calls raise.

Packed tensors are returned as ``torch.int32`` tensors holding the uint32 words
bit-for-bit (torch's uint32 dtype has too few kernels to be convenient); shape
``[bits][rows][packed_row_words(k)]`` (layout BMK').
"""
from __future__ import annotations

import ctypes
import os

import torch

__all__ = [
    "UNIPOLAR", "BIPOLAR", "SIGNED", "A_UNSIGNED", "A_BIPOLAR", "A_SIGNED", "ALGO_AUTO", "ALGO_POPC", "ALGO_POPC_LIT", "ALGO_GEMV", "ALGO_TC",
    "BitserialError", "library_path", "abi_version", "kernel_launches", "packed_row_words", "bitpack",
    "bitserial_dense", "bitserial_dense_i8", "bitserial_conv2d_nhwc", "bitserial_conv2d_nhwc_i8",
    "bitserial_conv2d_nhwc_host", "conv2d_workspace_bytes", "dense_workspace_bytes", "conv_out_extent",
    "bitserial_conv2d_nhwc_tc", "bitserial_dense_tc", "conv2d_tc_workspace_bytes", "dense_tc_workspace_bytes",
    "conv2d_tc_prepare_weights", "dense_tc_prepare_weights", "bitserial_conv2d_nhwc_tc_prepared",
    "bitserial_dense_tc_prepared", "bitserial_conv2d_nhwc_tc_i8", "bitserial_dense_tc_i8",
    "bitserial_conv2d_nhwc_tc_host", "conv2d_tc_weight_bytes", "dense_tc_weight_bytes", "TC_DEFAULT", "TC_I8",
    "TC_F4", "EXPORTED_SYMBOLS", "TcConvDesc", "bitserial_conv2d_nhwc_tc_group", "PackDesc", "bitpack_group",
    "bitserial_dense_tc_gather", "TcHostDesc", "bitserial_conv2d_nhwc_tc_host_group", "set_tuning", "get_tuning",
    "TUNE_TC_TILE_N", "TUNE_TC_EPILOGUE", "TUNE_TC_GROUP_SPLIT", "TUNE_TC_B_SLOTS", "TUNE_SMALL_KSPLIT",
    "TUNE_TCD_A_SRC", "TUNE_TCD_B_STREAM", "TUNE_TCD_MCAST", "ConvI8Desc",
    "bitserial_conv2d_nhwc_i8_group", "bitserial_dense_tc_multicast",
    "digit_row_bytes", "digitpack", "DigitPackDesc", "digitpack_group", "conv2d_tcd_weight_bytes",
    "dense_tcd_weight_bytes", "conv2d_tcd_prepare_weights", "dense_tcd_prepare_weights", "bitserial_conv2d_nhwc_tcd",
    "bitserial_dense_tcd", "TcdConvDesc", "bitserial_conv2d_nhwc_tcd_group",
    "tcw_act_bytes", "digitpack_win", "WinPackDesc", "digitpack_win_group", "conv2d_tcw_weight_bytes",
    "conv2d_tcw_prepare_weights", "bitserial_conv2d_nhwc_tcw", "TcwConvDesc", "bitserial_conv2d_nhwc_tcw_group",
]

UNIPOLAR, BIPOLAR, SIGNED = 0, 1, 2          # weight encodings (bs_encoding)
A_UNSIGNED, A_BIPOLAR, A_SIGNED = 0, 1, 2    # activation encodings (bs_a_encoding)
TC_DEFAULT, TC_I8, TC_F4 = 0, 1, 2  # bs_tc_format
ALGO_AUTO, ALGO_POPC, ALGO_POPC_LIT, ALGO_GEMV, ALGO_TC = 0, 1, 2, 3, 4
TUNE_TC_TILE_N, TUNE_TC_EPILOGUE, TUNE_TC_GROUP_SPLIT, TUNE_TC_B_SLOTS, TUNE_SMALL_KSPLIT = 0, 1, 2, 3, 4  # bs_tune_knob
TUNE_TCD_A_SRC, TUNE_TCD_B_STREAM, TUNE_TCD_MCAST = 5, 6, 7

_HERE = os.path.dirname(os.path.abspath(__file__))
# BITSERIAL_LIB selects an experiment build of the same library (A/B timing of compile-time
# variants in tools/); it must live under the repository's build/ directory.  Default: the
# in-tree product library.
_LIB_PATH = os.path.join(_HERE, "libbitserial.so")
if os.environ.get("BITSERIAL_LIB"):
    _alt = os.path.realpath(os.environ["BITSERIAL_LIB"])
    if not _alt.startswith(os.path.join(os.path.dirname(_HERE), "build") + os.sep):
        raise ImportError(f"BITSERIAL_LIB={_alt}: experiment builds must be under the repository's build/ directory")
    _LIB_PATH = _alt
_lib = None

EXPORTED_SYMBOLS = (
    "bs_abi_version", "bs_status_string", "bs_last_error", "bs_kernel_launches", "bs_packed_row_words", "bs_bitpack",
    "bs_bitpack_ex",
    "bs_bitserial_dense", "bs_bitserial_dense_ex", "bs_dense_workspace_bytes", "bs_bitserial_dense_i8",
    "bs_bitserial_conv2d_nhwc", "bs_bitserial_conv2d_nhwc_ex", "bs_conv2d_workspace_bytes",
    "bs_bitserial_conv2d_nhwc_i8", "bs_bitserial_conv2d_nhwc_host", "bs_conv2d_tc_workspace_bytes",
    "bs_bitserial_conv2d_nhwc_tc", "bs_dense_tc_workspace_bytes", "bs_bitserial_dense_tc",
    "bs_conv2d_tc_prepare_weights", "bs_dense_tc_prepare_weights", "bs_bitserial_conv2d_nhwc_tc_prepared",
    "bs_bitserial_dense_tc_prepared", "bs_bitserial_conv2d_nhwc_tc_i8", "bs_bitserial_dense_tc_i8",
    "bs_bitserial_conv2d_nhwc_tc_host", "bs_conv2d_tc_weight_bytes", "bs_dense_tc_weight_bytes",
    "bs_bitserial_conv2d_nhwc_tc_group", "bs_bitpack_group", "bs_bitpack_group_ex", "bs_bitserial_dense_tc_prepared_gather",
    "bs_bitserial_conv2d_nhwc_tc_host_group", "bs_set_tuning", "bs_get_tuning", "bs_bitserial_conv2d_nhwc_i8_group",
    "bs_bitserial_dense_tc_prepared_multicast", "bs_digit_row_bytes", "bs_digitpack", "bs_digitpack_group",
    "bs_conv2d_tcd_weight_bytes", "bs_dense_tcd_weight_bytes", "bs_conv2d_tcd_prepare_weights",
    "bs_dense_tcd_prepare_weights", "bs_bitserial_conv2d_nhwc_tcd", "bs_bitserial_dense_tcd",
    "bs_bitserial_conv2d_nhwc_tcd_group", "bs_tcw_act_bytes", "bs_digitpack_win", "bs_digitpack_win_group",
    "bs_conv2d_tcw_weight_bytes", "bs_conv2d_tcw_prepare_weights", "bs_bitserial_conv2d_nhwc_tcw",
    "bs_bitserial_conv2d_nhwc_tcw_group",
)


class BitserialError(RuntimeError):
    pass


def library_path() -> str:
    return _LIB_PATH


def _load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(_LIB_PATH):
        raise BitserialError(f"{_LIB_PATH} is missing: build it with `python -m paper_1810_11066_b200.build` "
                             "(there is no CPU fallback)")
    lib = ctypes.CDLL(_LIB_PATH)
    P, I, L = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
    sig = {
        "bs_abi_version": ([], I),
        "bs_status_string": ([I], ctypes.c_char_p),
        "bs_last_error": ([], ctypes.c_char_p),
        "bs_kernel_launches": ([], L),
        "bs_packed_row_words": ([L], L),
        "bs_bitpack": ([P, P, L, L, I, P], I),
        "bs_bitpack_ex": ([P, P, L, L, I, I, P], I),
        "bs_bitserial_dense": ([P, I, P, I, I, P, L, L, L, P], I),
        "bs_bitserial_dense_ex": ([P, I, P, I, I, P, L, L, L, I, P], I),
        "bs_dense_workspace_bytes": ([L, L, I], L),
        "bs_bitserial_dense_i8": ([P, I, P, I, I, P, L, L, L, P, L, P], I),
        "bs_bitserial_conv2d_nhwc": ([P, I, P, I, I, P] + [I] * 11 + [P], I),
        "bs_bitserial_conv2d_nhwc_ex": ([P, I, P, I, I, P] + [I] * 11 + [I, P], I),
        "bs_conv2d_workspace_bytes": ([I, I, I, I, I], L),
        "bs_bitserial_conv2d_nhwc_i8": ([P, I, P, I, I, P] + [I] * 11 + [P, L, P], I),
        "bs_bitserial_conv2d_nhwc_host": ([P, I, P, I, I, P] + [I] * 11 + [P, P, P, L, P], I),
        "bs_conv2d_tc_workspace_bytes": ([I, I, I, I, I], L),
        "bs_bitserial_conv2d_nhwc_tc": ([P, I, P, I, I, P] + [I] * 11 + [P, L, P], I),
        "bs_dense_tc_workspace_bytes": ([L, L, I], L),
        "bs_bitserial_dense_tc": ([P, I, P, I, I, P, L, L, L, P, L, P], I),
        "bs_conv2d_tc_weight_bytes": ([I, I, I, I, I, I], L),
        "bs_dense_tc_weight_bytes": ([L, L, I, I], L),
        "bs_conv2d_tc_prepare_weights": ([P, I, I, I, I, I, I, I, P, L, P], I),
        "bs_dense_tc_prepare_weights": ([P, I, I, L, L, I, P, L, P], I),
        "bs_bitserial_conv2d_nhwc_tc_prepared": ([P, I, I, P, I, I, I, P] + [I] * 11 + [P], I),
        "bs_bitserial_dense_tc_prepared": ([P, I, I, P, I, I, I, P, L, L, L, P], I),
        "bs_bitserial_conv2d_nhwc_tc_i8": ([P, I, I, P, I, I, I, P] + [I] * 11 + [P, L, P], I),
        "bs_bitserial_dense_tc_i8": ([P, I, I, P, I, I, I, P, L, L, L, P, L, P], I),
        "bs_bitserial_conv2d_nhwc_tc_host": ([P, I, I, P, I, I, I, P] + [I] * 11 + [P, P, P, L, P], I),
        "bs_bitserial_conv2d_nhwc_tc_group": ([P, I, I, I, I, P], I),
        "bs_bitpack_group": ([P, I, I, P], I),
        "bs_bitpack_group_ex": ([P, I, I, I, P], I),
        "bs_bitserial_conv2d_nhwc_tc_host_group": ([P, I, I, I, I, P], I),
        "bs_bitserial_dense_tc_prepared_gather": ([P, I, I, P, I, I, I, P, P, I, L, L, L, P], I),
        "bs_set_tuning": ([I, I], I),
        "bs_bitserial_dense_tc_prepared_multicast": ([P, I, I, P, I, I, I, P, L, L, L, P], I),
        "bs_bitserial_conv2d_nhwc_i8_group": ([P, I, I, I, P], I),
        "bs_get_tuning": ([I], I),
        "bs_digit_row_bytes": ([L], L),
        "bs_digitpack": ([P, P, L, L, I, I, P], I),
        "bs_digitpack_group": ([P, I, I, I, P], I),
        "bs_conv2d_tcd_weight_bytes": ([I, I, I, I, I], L),
        "bs_dense_tcd_weight_bytes": ([L, L, I], L),
        "bs_conv2d_tcd_prepare_weights": ([P, I, I, I, I, I, I, P, L, P], I),
        "bs_dense_tcd_prepare_weights": ([P, I, I, L, L, P, L, P], I),
        "bs_bitserial_conv2d_nhwc_tcd": ([P, I, I, P, I, I, P] + [I] * 11 + [P], I),
        "bs_bitserial_dense_tcd": ([P, I, I, P, I, I, P, L, L, L, P], I),
        "bs_bitserial_conv2d_nhwc_tcd_group": ([P, I, I, I, P], I),
        "bs_tcw_act_bytes": ([I] * 10, L),
        "bs_digitpack_win": ([P, P, L] + [I] * 11 + [P], I),
        "bs_digitpack_win_group": ([P, I, I, I, P], I),
        "bs_conv2d_tcw_weight_bytes": ([I, I, I, I, I], L),
        "bs_conv2d_tcw_prepare_weights": ([P, I, I, I, I, I, I, P, L, P], I),
        "bs_bitserial_conv2d_nhwc_tcw": ([P, I, I, P, I, I, P] + [I] * 11 + [P], I),
        "bs_bitserial_conv2d_nhwc_tcw_group": ([P, I, I, I, P], I),
    }
    for name, (args, res) in sig.items():
        if os.environ.get("BITSERIAL_LIB") and not hasattr(lib, name):
            continue  # an older experimental build (A/B timing) may lack newer entry points
        f = getattr(lib, name)
        f.argtypes, f.restype = args, res
    _lib = lib
    return lib


def _check(status: int):
    if status != 0:
        lib = _load()
        raise BitserialError(f"{lib.bs_status_string(status).decode()}: {lib.bs_last_error().decode()}")


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dev(t: torch.Tensor, name: str, dtype):
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise BitserialError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise BitserialError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise BitserialError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr())


def abi_version() -> int:
    return int(_load().bs_abi_version())


def kernel_launches() -> int:
    """Kernels launched by libbitserial.so so far in this process (bs_kernel_launches)."""
    return int(_load().bs_kernel_launches())


def set_tuning(knob: int, value: int) -> None:
    """bs_set_tuning: a process-wide launch-configuration knob (TUNE_*; 0 = library choice)."""
    _check(_load().bs_set_tuning(int(knob), int(value)))


def get_tuning(knob: int) -> int:
    return int(_load().bs_get_tuning(int(knob)))


def packed_row_words(k: int) -> int:
    return int(_load().bs_packed_row_words(int(k)))


def conv_out_extent(size: int, k: int, stride: int, pad: int) -> int:
    span = size + 2 * pad - k
    return span // stride + 1 if span >= 0 else 0


def dense_workspace_bytes(m: int, k: int, a_bits: int) -> int:
    return int(_load().bs_dense_workspace_bytes(m, k, a_bits))


def conv2d_workspace_bytes(n: int, h: int, w: int, c: int, a_bits: int) -> int:
    return int(_load().bs_conv2d_workspace_bytes(n, h, w, c, a_bits))


def bitpack(x: torch.Tensor, bits: int, out: torch.Tensor | None = None, stream=None, max_ctas: int = 0) -> torch.Tensor:
    """bs_bitpack(_ex): uint8 codes [rows][k] (or any shape, reduction axis last) ->
    int32-viewed uint32 words [bits][rows][packed_row_words(k)]; max_ctas > 0 caps the grid."""
    k = x.shape[-1]
    rows = x.numel() // k
    if out is None:
        out = torch.empty((bits, rows, packed_row_words(k)), dtype=torch.int32, device=x.device)
    _check(_load().bs_bitpack_ex(_dev(x, "x", torch.uint8), _dev(out, "out", torch.int32), rows, k, bits,
                                 int(max_ctas), _stream(stream)))
    return out


class PackDesc(ctypes.Structure):
    """bs_pack_desc (include/bitserial.h): one member of a grouped pack."""
    _fields_ = [("in_", ctypes.c_void_p), ("out", ctypes.c_void_p), ("rows", ctypes.c_int64), ("k", ctypes.c_int64)]


def bitpack_group(xs, bits, outs=None, stream=None, max_ctas=0):
    """bs_bitpack_group: bitpack every tensor of `xs` (uint8 codes, reduction axis last)
    at `bits` in one launch; returns the packed tensors (or fills `outs`)."""
    descs = (PackDesc * max(len(xs), 1))()
    res = []
    for i, x in enumerate(xs):
        k = x.shape[-1]
        rows = x.numel() // k
        out = outs[i] if outs is not None else torch.empty((bits, rows, packed_row_words(k)), dtype=torch.int32,
                                                            device=x.device)
        d = descs[i]
        d.in_ = _dev(x, "x", torch.uint8).value
        d.out = _dev(out, "out", torch.int32).value
        d.rows, d.k = rows, k
        res.append(out)
    _check(_load().bs_bitpack_group_ex(ctypes.cast(descs, ctypes.c_void_p), len(xs), bits, int(max_ctas),
                                       _stream(stream)))
    return res


def bitserial_dense(a_packed, a_bits, w_packed, w_bits, w_enc, m, n, k, out=None, algo=ALGO_AUTO, stream=None):
    """bs_bitserial_dense(_ex): out[m][n] = sum_k a[m][k] * value(w[n][k]) (int32)."""
    if out is None:
        out = torch.empty((m, n), dtype=torch.int32, device=a_packed.device)
    _check(_load().bs_bitserial_dense_ex(_dev(a_packed, "a_packed", torch.int32), a_bits,
                                         _dev(w_packed, "w_packed", torch.int32), w_bits, int(w_enc),
                                         _dev(out, "out", torch.int32), m, n, k, int(algo), _stream(stream)))
    return out


def bitserial_dense_i8(a, a_bits, w_packed, w_bits, w_enc, n, out=None, workspace=None, stream=None):
    """bs_bitserial_dense_i8: raw uint8 activation codes a [m][k] packed inside the call."""
    m, k = a.shape
    if out is None:
        out = torch.empty((m, n), dtype=torch.int32, device=a.device)
    need = dense_workspace_bytes(m, k, a_bits)
    if workspace is None:
        workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=a.device)
    _check(_load().bs_bitserial_dense_i8(_dev(a, "a", torch.uint8), a_bits, _dev(w_packed, "w_packed", torch.int32),
                                         w_bits, int(w_enc), _dev(out, "out", torch.int32), m, n, k,
                                         _dev(workspace, "workspace", torch.uint8), workspace.numel(),
                                         _stream(stream)))
    return out


def _conv_geom(n, h, w, kh, kw, stride, pad):
    sh, sw = (stride, stride) if isinstance(stride, int) else stride
    ph, pw = (pad, pad) if isinstance(pad, int) else pad
    return sh, sw, ph, pw, conv_out_extent(h, kh, sh, ph), conv_out_extent(w, kw, sw, pw)


def bitserial_conv2d_nhwc(act_packed, a_bits, w_packed, w_bits, w_enc, n, h, w, c, oc, kh, kw,
                          stride=1, pad=0, out=None, algo=ALGO_AUTO, stream=None):
    """bs_bitserial_conv2d_nhwc(_ex): packed NHWC activations x packed OHWI weights ->
    int32 NHWC [n][oh][ow][oc]."""
    sh, sw, ph, pw, oh, ow = _conv_geom(n, h, w, kh, kw, stride, pad)
    if out is None:
        out = torch.empty((n, max(oh, 0), max(ow, 0), oc), dtype=torch.int32, device=act_packed.device)
    _check(_load().bs_bitserial_conv2d_nhwc_ex(_dev(act_packed, "act_packed", torch.int32), a_bits,
                                               _dev(w_packed, "w_packed", torch.int32), w_bits, int(w_enc),
                                               _dev(out, "out", torch.int32), n, h, w, c, oc, kh, kw, sh, sw, ph, pw,
                                               int(algo), _stream(stream)))
    return out


def bitserial_conv2d_nhwc_i8(act, a_bits, w_packed, w_bits, w_enc, oc, kh, kw, stride=1, pad=0,
                             out=None, workspace=None, stream=None):
    """bs_bitserial_conv2d_nhwc_i8: raw uint8 NHWC activations [n][h][w][c], packed
    inside the call (the timed activation packing of PAPER.md:715)."""
    n, h, w, c = act.shape
    sh, sw, ph, pw, oh, ow = _conv_geom(n, h, w, kh, kw, stride, pad)
    if out is None:
        out = torch.empty((n, max(oh, 0), max(ow, 0), oc), dtype=torch.int32, device=act.device)
    need = conv2d_workspace_bytes(n, h, w, c, a_bits)
    if workspace is None:
        workspace = torch.empty(max(need, 16), dtype=torch.uint8, device=act.device)
    _check(_load().bs_bitserial_conv2d_nhwc_i8(_dev(act, "act", torch.uint8), a_bits,
                                               _dev(w_packed, "w_packed", torch.int32), w_bits, int(w_enc),
                                               _dev(out, "out", torch.int32), n, h, w, c, oc, kh, kw, sh, sw, ph, pw,
                                               _dev(workspace, "workspace", torch.uint8), workspace.numel(),
                                               _stream(stream)))
    return out


class ConvI8Desc(ctypes.Structure):
    """bs_conv_i8_desc (include/bitserial.h): one convolution of a one-launch small-problem group."""
    _fields_ = [("act", ctypes.c_void_p), ("w_packed", ctypes.c_void_p), ("out", ctypes.c_void_p),
                ("w_enc", ctypes.c_int)] + \
        [(f, ctypes.c_int) for f in ("n", "h", "w", "c", "oc", "kh", "kw", "stride_h", "stride_w", "pad_h", "pad_w")]


def bitserial_conv2d_nhwc_i8_group(convs, a_bits, w_bits, stream=None):
    """bs_bitserial_conv2d_nhwc_i8_group: several convolutions from raw uint8 NHWC codes in
    one launch (packing fused; the batch-1 latency path).  `convs`: dicts with act (uint8
    [n][h][w][c]), w_packed, w_enc, oc, kh, kw and optional stride, pad, out.  Returns the
    outputs in order."""
    descs = (ConvI8Desc * max(len(convs), 1))()
    outs = []
    for i, cv in enumerate(convs):
        act = cv["act"]
        n, h, w, c = act.shape
        sh, sw, ph, pw, oh, ow = _conv_geom(n, h, w, cv["kh"], cv["kw"], cv.get("stride", 1), cv.get("pad", 0))
        out = cv.get("out")
        if out is None:
            out = torch.empty((n, max(oh, 0), max(ow, 0), cv["oc"]), dtype=torch.int32, device=act.device)
        d = descs[i]
        d.act = _dev(act, "act", torch.uint8).value
        d.w_packed = _dev(cv["w_packed"], "w_packed", torch.int32).value
        d.out = _dev(out, "out", torch.int32).value
        d.w_enc = int(cv.get("w_enc", UNIPOLAR))
        d.n, d.h, d.w, d.c, d.oc, d.kh, d.kw = n, h, w, c, cv["oc"], cv["kh"], cv["kw"]
        d.stride_h, d.stride_w, d.pad_h, d.pad_w = sh, sw, ph, pw
        outs.append(out)
    _check(_load().bs_bitserial_conv2d_nhwc_i8_group(ctypes.cast(descs, ctypes.c_void_p), len(convs), a_bits, w_bits,
                                                     _stream(stream)))
    return outs


def conv2d_tc_workspace_bytes(oc, kh, kw, c, w_bits) -> int:
    return int(_load().bs_conv2d_tc_workspace_bytes(oc, kh, kw, c, w_bits))


def dense_tc_workspace_bytes(n, k, w_bits) -> int:
    return int(_load().bs_dense_tc_workspace_bytes(n, k, w_bits))


def bitserial_conv2d_nhwc_tc(act_packed, a_bits, w_packed, w_bits, w_enc, n, h, w, c, oc, kh, kw,
                             stride=1, pad=0, out=None, workspace=None, stream=None):
    """bs_bitserial_conv2d_nhwc_tc: the tensor-core bitserial conv (tcgen05, kind::i8)."""
    sh, sw, ph, pw, oh, ow = _conv_geom(n, h, w, kh, kw, stride, pad)
    if out is None:
        out = torch.empty((n, max(oh, 0), max(ow, 0), oc), dtype=torch.int32, device=act_packed.device)
    if workspace is None:
        workspace = torch.empty(max(16, conv2d_tc_workspace_bytes(oc, kh, kw, c, w_bits)), dtype=torch.uint8,
                                device=act_packed.device)
    _check(_load().bs_bitserial_conv2d_nhwc_tc(_dev(act_packed, "act_packed", torch.int32), a_bits,
                                               _dev(w_packed, "w_packed", torch.int32), w_bits, int(w_enc),
                                               _dev(out, "out", torch.int32), n, h, w, c, oc, kh, kw, sh, sw, ph, pw,
                                               _dev(workspace, "workspace", torch.uint8), workspace.numel(),
                                               _stream(stream)))
    return out


def bitserial_dense_tc(a_packed, a_bits, w_packed, w_bits, w_enc, m, n, k, out=None, workspace=None, stream=None):
    """bs_bitserial_dense_tc: the tensor-core bitserial dense product (tcgen05, kind::i8)."""
    if out is None:
        out = torch.empty((m, n), dtype=torch.int32, device=a_packed.device)
    if workspace is None:
        workspace = torch.empty(max(16, dense_tc_workspace_bytes(n, k, w_bits)), dtype=torch.uint8,
                                device=a_packed.device)
    _check(_load().bs_bitserial_dense_tc(_dev(a_packed, "a_packed", torch.int32), a_bits,
                                         _dev(w_packed, "w_packed", torch.int32), w_bits, int(w_enc),
                                         _dev(out, "out", torch.int32), m, n, k,
                                         _dev(workspace, "workspace", torch.uint8), workspace.numel(),
                                         _stream(stream)))
    return out


def conv2d_tc_weight_bytes(oc, kh, kw, c, w_bits, tc_format=TC_DEFAULT) -> int:
    return int(_load().bs_conv2d_tc_weight_bytes(oc, kh, kw, c, w_bits, int(tc_format)))


def dense_tc_weight_bytes(n, k, w_bits, tc_format=TC_DEFAULT) -> int:
    return int(_load().bs_dense_tc_weight_bytes(n, k, w_bits, int(tc_format)))


def conv2d_tc_prepare_weights(w_packed, w_bits, w_enc, oc, kh, kw, c, tc_format=TC_DEFAULT, out=None, stream=None):
    """bs_conv2d_tc_prepare_weights: packed OHWI weights -> prepared (expanded) tensor-core
    weights for `tc_format` (offline, like weight packing)."""
    if out is None:
        out = torch.empty(max(16, conv2d_tc_weight_bytes(oc, kh, kw, c, w_bits, tc_format)), dtype=torch.int8,
                          device=w_packed.device)
    _check(_load().bs_conv2d_tc_prepare_weights(_dev(w_packed, "w_packed", torch.int32), w_bits, int(w_enc), oc, kh, kw,
                                                c, int(tc_format), _dev(out, "w_tc", torch.int8), out.numel(),
                                                _stream(stream)))
    return out


def dense_tc_prepare_weights(w_packed, w_bits, w_enc, n, k, tc_format=TC_DEFAULT, out=None, stream=None):
    """bs_dense_tc_prepare_weights: packed [n][k] weights -> prepared tensor-core weights."""
    if out is None:
        out = torch.empty(max(16, dense_tc_weight_bytes(n, k, w_bits, tc_format)), dtype=torch.int8,
                          device=w_packed.device)
    _check(_load().bs_dense_tc_prepare_weights(_dev(w_packed, "w_packed", torch.int32), w_bits, int(w_enc), n, k,
                                               int(tc_format), _dev(out, "w_tc", torch.int8), out.numel(),
                                               _stream(stream)))
    return out


def bitserial_conv2d_nhwc_tc_prepared(act_packed, a_bits, w_tc, w_bits, n, h, w, c, oc, kh, kw, stride=1, pad=0,
                                      out=None, tc_format=TC_DEFAULT, stream=None, a_enc=A_UNSIGNED, w_enc=UNIPOLAR):
    """bs_bitserial_conv2d_nhwc_tc_prepared: packed activations x prepared weights -> int32 NHWC
    (a_enc: activation encoding; w_enc: the encoding the weights were prepared with)."""
    sh, sw, ph, pw, oh, ow = _conv_geom(n, h, w, kh, kw, stride, pad)
    if out is None:
        out = torch.empty((n, max(oh, 0), max(ow, 0), oc), dtype=torch.int32, device=act_packed.device)
    _check(_load().bs_bitserial_conv2d_nhwc_tc_prepared(
        _dev(act_packed, "act_packed", torch.int32), a_bits, int(a_enc), _dev(w_tc, "w_tc", torch.int8), w_bits,
        int(w_enc), int(tc_format),
        _dev(out, "out", torch.int32), n, h, w, c, oc, kh, kw, sh, sw, ph, pw, _stream(stream)))
    return out


class TcConvDesc(ctypes.Structure):
    """bs_tc_conv_desc (include/bitserial.h): one member of a grouped tensor-core launch."""
    _fields_ = [("act_packed", ctypes.c_void_p), ("w_tc", ctypes.c_void_p), ("out", ctypes.c_void_p),
                ("a_enc", ctypes.c_int), ("w_enc", ctypes.c_int)] + \
        [(f, ctypes.c_int) for f in ("n", "h", "w", "c", "oc", "kh", "kw", "stride_h", "stride_w", "pad_h", "pad_w")]


def bitserial_conv2d_nhwc_tc_group(convs, a_bits, w_bits, tc_format=TC_DEFAULT, stream=None):
    """bs_bitserial_conv2d_nhwc_tc_group: several prepared-weight convolutions of one
    precision in one persistent launch.  `convs` is a sequence of dicts with the keys of
    bitserial_conv2d_nhwc_tc_prepared (act_packed, w_tc, n, h, w, c, oc, kh, kw and
    optional stride, pad, out, a_enc, w_enc).  Returns the output tensors in order."""
    descs = (TcConvDesc * max(len(convs), 1))()
    outs = []
    for i, cv in enumerate(convs):
        n, h, w, c, oc, kh, kw = (cv[k] for k in ("n", "h", "w", "c", "oc", "kh", "kw"))
        sh, sw, ph, pw, oh, ow = _conv_geom(n, h, w, kh, kw, cv.get("stride", 1), cv.get("pad", 0))
        out = cv.get("out")
        if out is None:
            out = torch.empty((n, max(oh, 0), max(ow, 0), oc), dtype=torch.int32, device=cv["act_packed"].device)
        d = descs[i]
        d.act_packed = _dev(cv["act_packed"], "act_packed", torch.int32).value
        d.w_tc = _dev(cv["w_tc"], "w_tc", torch.int8).value
        d.out = _dev(out, "out", torch.int32).value
        d.a_enc, d.w_enc = int(cv.get("a_enc", A_UNSIGNED)), int(cv.get("w_enc", UNIPOLAR))
        d.n, d.h, d.w, d.c, d.oc, d.kh, d.kw = n, h, w, c, oc, kh, kw
        d.stride_h, d.stride_w, d.pad_h, d.pad_w = sh, sw, ph, pw
        outs.append(out)
    _check(_load().bs_bitserial_conv2d_nhwc_tc_group(ctypes.cast(descs, ctypes.c_void_p), len(convs), a_bits,
                                                     w_bits, int(tc_format), _stream(stream)))
    return outs


def bitserial_dense_tc_prepared(a_packed, a_bits, w_tc, w_bits, m, n, k, out=None, tc_format=TC_DEFAULT,
                                stream=None, a_enc=A_UNSIGNED, w_enc=UNIPOLAR):
    """bs_bitserial_dense_tc_prepared: packed activations x prepared weights -> int32 [m][n]."""
    if out is None:
        out = torch.empty((m, n), dtype=torch.int32, device=a_packed.device)
    _check(_load().bs_bitserial_dense_tc_prepared(_dev(a_packed, "a_packed", torch.int32), a_bits, int(a_enc),
                                                  _dev(w_tc, "w_tc", torch.int8), w_bits, int(w_enc), int(tc_format),
                                                  _dev(out, "out", torch.int32), m, n, k, _stream(stream)))
    return out


class TcHostDesc(ctypes.Structure):
    """bs_tc_host_desc (include/bitserial.h): one layer of a pipelined host-buffer call."""
    _fields_ = [("act_host", ctypes.c_void_p), ("out_host", ctypes.c_void_p), ("act_dev", ctypes.c_void_p),
                ("packed_dev", ctypes.c_void_p), ("out_dev", ctypes.c_void_p), ("w_tc", ctypes.c_void_p),
                ("a_enc", ctypes.c_int), ("w_enc", ctypes.c_int)] + \
        [(f, ctypes.c_int) for f in ("n", "h", "w", "c", "oc", "kh", "kw", "stride_h", "stride_w", "pad_h", "pad_w")]


def _host_ptr(t: torch.Tensor, name: str, dtype):
    if not isinstance(t, torch.Tensor) or t.device.type != "cpu" or t.dtype != dtype or not t.is_contiguous():
        raise BitserialError(f"{name} must be a contiguous CPU {dtype} tensor")
    return t.data_ptr()


def bitserial_conv2d_nhwc_tc_host_group(layers, a_bits, w_bits, tc_format=TC_DEFAULT, stream=None):
    """bs_bitserial_conv2d_nhwc_tc_host_group: every layer host -> device -> pack -> conv ->
    host, pipelined over three streams.  `layers`: dicts with act_host (uint8 NHWC, pinned),
    out_host (int32, pinned), act_dev, packed_dev (int32 workspace), out_dev, w_tc, oc, kh,
    kw and optional stride, pad, a_enc, w_enc.  Returns the out_host tensors."""
    descs = (TcHostDesc * max(len(layers), 1))()
    for i, ly in enumerate(layers):
        n, h, w, c = ly["act_host"].shape
        sh, sw, ph, pw, _, _ = _conv_geom(n, h, w, ly["kh"], ly["kw"], ly.get("stride", 1), ly.get("pad", 0))
        d = descs[i]
        d.act_host = _host_ptr(ly["act_host"], "act_host", torch.uint8)
        d.out_host = _host_ptr(ly["out_host"], "out_host", torch.int32)
        d.act_dev = _dev(ly["act_dev"], "act_dev", torch.uint8).value
        d.packed_dev = _dev(ly["packed_dev"], "packed_dev", ly["packed_dev"].dtype).value
        d.out_dev = _dev(ly["out_dev"], "out_dev", torch.int32).value
        d.w_tc = _dev(ly["w_tc"], "w_tc", torch.int8).value
        d.a_enc, d.w_enc = int(ly.get("a_enc", A_UNSIGNED)), int(ly.get("w_enc", UNIPOLAR))
        d.n, d.h, d.w, d.c, d.oc, d.kh, d.kw = n, h, w, c, ly["oc"], ly["kh"], ly["kw"]
        d.stride_h, d.stride_w, d.pad_h, d.pad_w = sh, sw, ph, pw
    _check(_load().bs_bitserial_conv2d_nhwc_tc_host_group(ctypes.cast(descs, ctypes.c_void_p), len(layers), a_bits,
                                                          w_bits, int(tc_format), _stream(stream)))
    return [ly["out_host"] for ly in layers]


def bitserial_dense_tc_gather(a_packed, a_bits, w_tc, w_bits, m, n, k, out, peers, tc_format=TC_DEFAULT,
                              stream=None, a_enc=A_UNSIGNED, w_enc=UNIPOLAR):
    """bs_bitserial_dense_tc_prepared_gather: this rank's [m][n] row block of C written to
    `out` and, from the same staged tiles, to every peer block in `peers` (CUDA tensors —
    e.g. other ranks' symmetric-memory buffers — or raw device addresses)."""
    ptrs = (ctypes.c_void_p * max(len(peers), 1))()
    for i, p in enumerate(peers):
        ptrs[i] = _dev(p, "peer", torch.int32).value if isinstance(p, torch.Tensor) else int(p)
    _check(_load().bs_bitserial_dense_tc_prepared_gather(
        _dev(a_packed, "a_packed", torch.int32), a_bits, int(a_enc), _dev(w_tc, "w_tc", torch.int8), w_bits,
        int(w_enc), int(tc_format), _dev(out, "out", torch.int32), ctypes.cast(ptrs, ctypes.c_void_p), len(peers),
        m, n, k, _stream(stream)))
    return out


def bitserial_dense_tc_multicast(a_packed, a_bits, w_tc, w_bits, m, n, k, out_mc, tc_format=TC_DEFAULT, stream=None,
                                 a_enc=A_UNSIGNED, w_enc=UNIPOLAR):
    """bs_bitserial_dense_tc_prepared_multicast: this rank's [m][n] row block of C stored once,
    with multimem.st, to `out_mc` — the multicast (NVLS) device address (int) of that block."""
    _check(_load().bs_bitserial_dense_tc_prepared_multicast(
        _dev(a_packed, "a_packed", torch.int32), a_bits, int(a_enc), _dev(w_tc, "w_tc", torch.int8), w_bits,
        int(w_enc), int(tc_format), ctypes.c_void_p(int(out_mc)), m, n, k, _stream(stream)))


def bitserial_conv2d_nhwc_tc_i8(act, a_bits, w_tc, w_bits, oc, kh, kw, stride=1, pad=0, out=None, workspace=None,
                                tc_format=TC_DEFAULT, stream=None, a_enc=A_UNSIGNED, w_enc=UNIPOLAR):
    """bs_bitserial_conv2d_nhwc_tc_i8: raw uint8 NHWC activations packed inside the call,
    then the tensor-core conv on prepared weights (the timed step)."""
    n, h, w, c = act.shape
    sh, sw, ph, pw, oh, ow = _conv_geom(n, h, w, kh, kw, stride, pad)
    if out is None:
        out = torch.empty((n, max(oh, 0), max(ow, 0), oc), dtype=torch.int32, device=act.device)
    if workspace is None:
        workspace = torch.empty(max(conv2d_workspace_bytes(n, h, w, c, a_bits), 16), dtype=torch.uint8,
                                device=act.device)
    _check(_load().bs_bitserial_conv2d_nhwc_tc_i8(
        _dev(act, "act", torch.uint8), a_bits, int(a_enc), _dev(w_tc, "w_tc", torch.int8), w_bits, int(w_enc),
        int(tc_format), _dev(out, "out", torch.int32),
        n, h, w, c, oc, kh, kw, sh, sw, ph, pw, _dev(workspace, "workspace", torch.uint8), workspace.numel(),
        _stream(stream)))
    return out


def bitserial_dense_tc_i8(a, a_bits, w_tc, w_bits, n, out=None, workspace=None, tc_format=TC_DEFAULT, stream=None,
                          a_enc=A_UNSIGNED, w_enc=UNIPOLAR):
    """bs_bitserial_dense_tc_i8: raw uint8 activations [m][k] packed inside the call, then
    the tensor-core dense product on prepared weights."""
    m, k = a.shape
    if out is None:
        out = torch.empty((m, n), dtype=torch.int32, device=a.device)
    if workspace is None:
        workspace = torch.empty(max(dense_workspace_bytes(m, k, a_bits), 16), dtype=torch.uint8, device=a.device)
    _check(_load().bs_bitserial_dense_tc_i8(_dev(a, "a", torch.uint8), a_bits, int(a_enc),
                                            _dev(w_tc, "w_tc", torch.int8), w_bits, int(w_enc),
                                            int(tc_format), _dev(out, "out", torch.int32), m, n, k,
                                            _dev(workspace, "workspace", torch.uint8), workspace.numel(),
                                            _stream(stream)))
    return out


def bitserial_conv2d_nhwc_tc_host(act_host, a_bits, w_tc, w_bits, oc, kh, kw, stride, pad, out_host, act_dev, out_dev,
                                  workspace, tc_format=TC_DEFAULT, stream=None, a_enc=A_UNSIGNED, w_enc=UNIPOLAR):
    """bs_bitserial_conv2d_nhwc_tc_host: the e2e path (host in, host out) on the tensor-core kernel."""
    if act_host.device.type != "cpu" or out_host.device.type != "cpu":
        raise BitserialError("act_host/out_host must be CPU tensors")
    if not (act_host.is_contiguous() and out_host.is_contiguous()):
        raise BitserialError("host buffers must be contiguous")
    n, h, w, c = act_host.shape
    sh, sw, ph, pw, _, _ = _conv_geom(n, h, w, kh, kw, stride, pad)
    _check(_load().bs_bitserial_conv2d_nhwc_tc_host(
        ctypes.c_void_p(act_host.data_ptr()), a_bits, int(a_enc), _dev(w_tc, "w_tc", torch.int8), w_bits, int(w_enc),
        int(tc_format),
        ctypes.c_void_p(out_host.data_ptr()), n, h, w, c, oc, kh, kw, sh, sw, ph, pw,
        _dev(act_dev, "act_dev", torch.uint8), _dev(out_dev, "out_dev", torch.int32),
        _dev(workspace, "workspace", torch.uint8), workspace.numel(), _stream(stream)))
    return out_host


def bitserial_conv2d_nhwc_host(act_host, a_bits, w_packed, w_bits, w_enc, oc, kh, kw, stride, pad,
                               out_host, act_dev, out_dev, workspace, stream=None):
    """bs_bitserial_conv2d_nhwc_host: host uint8 NHWC in, host int32 NHWC out; copies,
    packs, convolves and synchronizes inside the call (the e2e path)."""
    if act_host.device.type != "cpu" or out_host.device.type != "cpu":
        raise BitserialError("act_host/out_host must be CPU tensors")
    if not (act_host.is_contiguous() and out_host.is_contiguous()):
        raise BitserialError("host buffers must be contiguous")
    n, h, w, c = act_host.shape
    sh, sw, ph, pw, _, _ = _conv_geom(n, h, w, kh, kw, stride, pad)
    _check(_load().bs_bitserial_conv2d_nhwc_host(
        ctypes.c_void_p(act_host.data_ptr()), a_bits, _dev(w_packed, "w_packed", torch.int32), w_bits, int(w_enc),
        ctypes.c_void_p(out_host.data_ptr()), n, h, w, c, oc, kh, kw, sh, sw, ph, pw,
        _dev(act_dev, "act_dev", torch.uint8), _dev(out_dev, "out_dev", torch.int32),
        _dev(workspace, "workspace", torch.uint8), workspace.numel(), _stream(stream)))
    return out_host


# ---------------------------------------------------------------- digit-packed path
def digit_row_bytes(k: int) -> int:
    """bs_digit_row_bytes: bytes per digit-packed row (16 * packed_row_words(k))."""
    return int(_load().bs_digit_row_bytes(int(k)))


def digitpack(x: torch.Tensor, bits: int, enc: int = A_UNSIGNED, out: torch.Tensor | None = None,
              stream=None) -> torch.Tensor:
    """bs_digitpack: uint8 codes [rows][k] (reduction axis last) -> uint8 E2M1 digit fields
    [ceil(bits/2)][rows][digit_row_bytes(k)] (two bit planes per 4-bit field, R24)."""
    k = x.shape[-1]
    rows = x.numel() // k
    if out is None:
        out = torch.empty(((bits + 1) // 2, rows, digit_row_bytes(k)), dtype=torch.uint8, device=x.device)
    _check(_load().bs_digitpack(_dev(x, "x", torch.uint8), _dev(out, "out", torch.uint8), rows, k, bits, int(enc),
                                _stream(stream)))
    return out


class DigitPackDesc(ctypes.Structure):
    """bs_digit_pack_desc (include/bitserial.h): one member of a grouped digit pack."""
    _fields_ = [("in_", ctypes.c_void_p), ("out", ctypes.c_void_p), ("rows", ctypes.c_int64), ("k", ctypes.c_int64)]


def digitpack_group(xs, bits, enc=A_UNSIGNED, outs=None, stream=None):
    """bs_digitpack_group: digit-pack every tensor of `xs` in one launch."""
    descs = (DigitPackDesc * max(len(xs), 1))()
    res = []
    for i, x in enumerate(xs):
        k = x.shape[-1]
        rows = x.numel() // k
        out = outs[i] if outs is not None else torch.empty(((bits + 1) // 2, rows, digit_row_bytes(k)),
                                                            dtype=torch.uint8, device=x.device)
        d = descs[i]
        d.in_ = _dev(x, "x", torch.uint8).value
        d.out = _dev(out, "out", torch.uint8).value
        d.rows, d.k = rows, k
        res.append(out)
    _check(_load().bs_digitpack_group(ctypes.cast(descs, ctypes.c_void_p), len(xs), bits, int(enc), _stream(stream)))
    return res


def conv2d_tcd_weight_bytes(oc, kh, kw, c, w_bits) -> int:
    return int(_load().bs_conv2d_tcd_weight_bytes(oc, kh, kw, c, w_bits))


def dense_tcd_weight_bytes(n, k, w_bits) -> int:
    return int(_load().bs_dense_tcd_weight_bytes(n, k, w_bits))


def conv2d_tcd_prepare_weights(w_packed, w_bits, w_enc, oc, kh, kw, c, out=None, stream=None):
    """bs_conv2d_tcd_prepare_weights: packed OHWI weight planes -> weight digits (offline)."""
    if out is None:
        out = torch.empty(max(16, conv2d_tcd_weight_bytes(oc, kh, kw, c, w_bits)), dtype=torch.uint8,
                          device=w_packed.device)
    _check(_load().bs_conv2d_tcd_prepare_weights(_dev(w_packed, "w_packed", torch.int32), w_bits, int(w_enc), oc, kh,
                                                 kw, c, _dev(out, "w_dig", torch.uint8), out.numel(), _stream(stream)))
    return out


def dense_tcd_prepare_weights(w_packed, w_bits, w_enc, n, k, out=None, stream=None):
    """bs_dense_tcd_prepare_weights: packed [n][k] weight planes -> weight digits (offline)."""
    if out is None:
        out = torch.empty(max(16, dense_tcd_weight_bytes(n, k, w_bits)), dtype=torch.uint8, device=w_packed.device)
    _check(_load().bs_dense_tcd_prepare_weights(_dev(w_packed, "w_packed", torch.int32), w_bits, int(w_enc), n, k,
                                                _dev(out, "w_dig", torch.uint8), out.numel(), _stream(stream)))
    return out


def bitserial_conv2d_nhwc_tcd(act_dig, a_bits, w_dig, w_bits, n, h, w, c, oc, kh, kw, stride=1, pad=0, out=None,
                              a_enc=A_UNSIGNED, w_enc=UNIPOLAR, stream=None):
    """bs_bitserial_conv2d_nhwc_tcd: digit-packed activations x weight digits -> int32 NHWC."""
    sh, sw, ph, pw, oh, ow = _conv_geom(n, h, w, kh, kw, stride, pad)
    if out is None:
        out = torch.empty((n, max(oh, 0), max(ow, 0), oc), dtype=torch.int32, device=act_dig.device)
    _check(_load().bs_bitserial_conv2d_nhwc_tcd(
        _dev(act_dig, "act_dig", torch.uint8), a_bits, int(a_enc), _dev(w_dig, "w_dig", torch.uint8), w_bits,
        int(w_enc), _dev(out, "out", torch.int32), n, h, w, c, oc, kh, kw, sh, sw, ph, pw, _stream(stream)))
    return out


def bitserial_dense_tcd(a_dig, a_bits, w_dig, w_bits, m, n, k, out=None, a_enc=A_UNSIGNED, w_enc=UNIPOLAR,
                        stream=None):
    """bs_bitserial_dense_tcd: digit-packed activations [D][m][..] x weight digits -> int32 [m][n]."""
    if out is None:
        out = torch.empty((m, n), dtype=torch.int32, device=a_dig.device)
    _check(_load().bs_bitserial_dense_tcd(_dev(a_dig, "a_dig", torch.uint8), a_bits, int(a_enc),
                                          _dev(w_dig, "w_dig", torch.uint8), w_bits, int(w_enc),
                                          _dev(out, "out", torch.int32), m, n, k, _stream(stream)))
    return out


class TcdConvDesc(ctypes.Structure):
    """bs_tcd_conv_desc (include/bitserial.h): one member of a grouped digit-path launch."""
    _fields_ = [("act_dig", ctypes.c_void_p), ("w_dig", ctypes.c_void_p), ("out", ctypes.c_void_p),
                ("a_enc", ctypes.c_int), ("w_enc", ctypes.c_int)] + \
        [(f, ctypes.c_int) for f in ("n", "h", "w", "c", "oc", "kh", "kw", "stride_h", "stride_w", "pad_h", "pad_w")]


def bitserial_conv2d_nhwc_tcd_group(convs, a_bits, w_bits, stream=None):
    """bs_bitserial_conv2d_nhwc_tcd_group: several digit-path convolutions of one precision in
    one launch.  `convs`: dicts with act_dig, w_dig, n, h, w, c, oc, kh, kw and optional
    stride, pad, out, a_enc, w_enc.  Returns the outputs in order."""
    descs = (TcdConvDesc * max(len(convs), 1))()
    outs = []
    for i, cv in enumerate(convs):
        n, h, w, c, oc, kh, kw = (cv[k] for k in ("n", "h", "w", "c", "oc", "kh", "kw"))
        sh, sw, ph, pw, oh, ow = _conv_geom(n, h, w, kh, kw, cv.get("stride", 1), cv.get("pad", 0))
        out = cv.get("out")
        if out is None:
            out = torch.empty((n, max(oh, 0), max(ow, 0), oc), dtype=torch.int32, device=cv["act_dig"].device)
        d = descs[i]
        d.act_dig = _dev(cv["act_dig"], "act_dig", torch.uint8).value
        d.w_dig = _dev(cv["w_dig"], "w_dig", torch.uint8).value
        d.out = _dev(out, "out", torch.int32).value
        d.a_enc, d.w_enc = int(cv.get("a_enc", A_UNSIGNED)), int(cv.get("w_enc", UNIPOLAR))
        d.n, d.h, d.w, d.c, d.oc, d.kh, d.kw = n, h, w, c, oc, kh, kw
        d.stride_h, d.stride_w, d.pad_h, d.pad_w = sh, sw, ph, pw
        outs.append(out)
    _check(_load().bs_bitserial_conv2d_nhwc_tcd_group(ctypes.cast(descs, ctypes.c_void_p), len(convs), a_bits, w_bits,
                                                      _stream(stream)))
    return outs


# ---------------------------------------------------------------- window path (R26)
def tcw_act_bytes(n, h, w, c, kh, kw, stride, pad, bits) -> int:
    """bs_tcw_act_bytes: bytes of the window layout of an [n][h][w][c] input for this conv
    geometry (0 outside the layout's domain)."""
    ph, pw = (pad, pad) if isinstance(pad, int) else pad
    return int(_load().bs_tcw_act_bytes(n, h, w, c, kh, kw, int(stride), ph, pw, bits))


def digitpack_win(x: torch.Tensor, bits: int, kh: int, kw: int, stride: int = 1, pad=0, enc: int = A_UNSIGNED,
                  out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """bs_digitpack_win: uint8 NHWC codes [n][h][w][c] -> the window layout of the conv
    (kh x kw, stride, pad) as a flat uint8 tensor of bs_tcw_act_bytes bytes."""
    n, h, w, c = x.shape
    ph, pw = (pad, pad) if isinstance(pad, int) else pad
    nbytes = tcw_act_bytes(n, h, w, c, kh, kw, stride, (ph, pw), bits)
    if out is None:
        out = torch.empty(max(16, nbytes), dtype=torch.uint8, device=x.device)
    _check(_load().bs_digitpack_win(_dev(x, "x", torch.uint8), _dev(out, "out", torch.uint8), out.numel(), n, h, w, c,
                                    kh, kw, int(stride), ph, pw, bits, int(enc), _stream(stream)))
    return out


class WinPackDesc(ctypes.Structure):
    """bs_win_pack_desc (include/bitserial.h): one member of a grouped window-layout pack."""
    _fields_ = [("in_", ctypes.c_void_p), ("out", ctypes.c_void_p), ("out_bytes", ctypes.c_int64)] + \
        [(f, ctypes.c_int) for f in ("n", "h", "w", "c", "kh", "kw", "stride", "pad_h", "pad_w")]


def digitpack_win_group(items, bits, enc=A_UNSIGNED, outs=None, stream=None):
    """bs_digitpack_win_group: window-pack several NHWC tensors in one launch.  `items`:
    dicts with x, kh, kw and optional stride, pad.  Returns the flat layouts in order."""
    descs = (WinPackDesc * max(len(items), 1))()
    res = []
    for i, it in enumerate(items):
        x = it["x"]
        n, h, w, c = x.shape
        st = int(it.get("stride", 1))
        pad = it.get("pad", 0)
        ph, pw = (pad, pad) if isinstance(pad, int) else pad
        nbytes = tcw_act_bytes(n, h, w, c, it["kh"], it["kw"], st, (ph, pw), bits)
        out = outs[i] if outs is not None else torch.empty(max(16, nbytes), dtype=torch.uint8, device=x.device)
        d = descs[i]
        d.in_ = _dev(x, "x", torch.uint8).value
        d.out = _dev(out, "out", torch.uint8).value
        d.out_bytes = out.numel()
        d.n, d.h, d.w, d.c, d.kh, d.kw, d.stride, d.pad_h, d.pad_w = n, h, w, c, it["kh"], it["kw"], st, ph, pw
        res.append(out)
    _check(_load().bs_digitpack_win_group(ctypes.cast(descs, ctypes.c_void_p), len(items), bits, int(enc),
                                          _stream(stream)))
    return res


def conv2d_tcw_weight_bytes(oc, kh, kw, c, w_bits) -> int:
    return int(_load().bs_conv2d_tcw_weight_bytes(oc, kh, kw, c, w_bits))


def conv2d_tcw_prepare_weights(w_packed, w_bits, w_enc, oc, kh, kw, c, out=None, stream=None):
    """bs_conv2d_tcw_prepare_weights: packed OHWI weight planes -> window-path weight digits."""
    if out is None:
        out = torch.empty(max(16, conv2d_tcw_weight_bytes(oc, kh, kw, c, w_bits)), dtype=torch.uint8,
                          device=w_packed.device)
    _check(_load().bs_conv2d_tcw_prepare_weights(_dev(w_packed, "w_packed", torch.int32), w_bits, int(w_enc), oc, kh,
                                                 kw, c, _dev(out, "w_win", torch.uint8), out.numel(), _stream(stream)))
    return out


def bitserial_conv2d_nhwc_tcw(act_win, a_bits, w_win, w_bits, n, h, w, c, oc, kh, kw, stride=1, pad=0, out=None,
                              a_enc=A_UNSIGNED, w_enc=UNIPOLAR, stream=None):
    """bs_bitserial_conv2d_nhwc_tcw: window-layout activations x window-path weights -> int32 NHWC."""
    sh, sw, ph, pw, oh, ow = _conv_geom(n, h, w, kh, kw, stride, pad)
    if out is None:
        out = torch.empty((n, max(oh, 0), max(ow, 0), oc), dtype=torch.int32, device=act_win.device)
    _check(_load().bs_bitserial_conv2d_nhwc_tcw(
        _dev(act_win, "act_win", torch.uint8), a_bits, int(a_enc), _dev(w_win, "w_win", torch.uint8), w_bits,
        int(w_enc), _dev(out, "out", torch.int32), n, h, w, c, oc, kh, kw, sh, sw, ph, pw, _stream(stream)))
    return out


class TcwConvDesc(ctypes.Structure):
    """bs_tcw_conv_desc (include/bitserial.h): one member of a grouped window-path launch."""
    _fields_ = [("act_win", ctypes.c_void_p), ("w_win", ctypes.c_void_p), ("out", ctypes.c_void_p),
                ("a_enc", ctypes.c_int), ("w_enc", ctypes.c_int)] + \
        [(f, ctypes.c_int) for f in ("n", "h", "w", "c", "oc", "kh", "kw", "stride_h", "stride_w", "pad_h", "pad_w")]


def bitserial_conv2d_nhwc_tcw_group(convs, a_bits, w_bits, stream=None):
    """bs_bitserial_conv2d_nhwc_tcw_group: several window-path convolutions of one precision in
    one launch.  `convs`: dicts with act_win, w_win, n, h, w, c, oc, kh, kw and optional stride,
    pad, out, a_enc, w_enc.  Returns the outputs in order."""
    descs = (TcwConvDesc * max(len(convs), 1))()
    outs = []
    for i, cv in enumerate(convs):
        n, h, w, c, oc, kh, kw = (cv[k] for k in ("n", "h", "w", "c", "oc", "kh", "kw"))
        sh, sw, ph, pw, oh, ow = _conv_geom(n, h, w, kh, kw, cv.get("stride", 1), cv.get("pad", 0))
        out = cv.get("out")
        if out is None:
            out = torch.empty((n, max(oh, 0), max(ow, 0), oc), dtype=torch.int32, device=cv["act_win"].device)
        d = descs[i]
        d.act_win = _dev(cv["act_win"], "act_win", torch.uint8).value
        d.w_win = _dev(cv["w_win"], "w_win", torch.uint8).value
        d.out = _dev(out, "out", torch.int32).value
        d.a_enc, d.w_enc = int(cv.get("a_enc", A_UNSIGNED)), int(cv.get("w_enc", UNIPOLAR))
        d.n, d.h, d.w, d.c, d.oc, d.kh, d.kw = n, h, w, c, oc, kh, kw
        d.stride_h, d.stride_w, d.pad_h, d.pad_w = sh, sw, ph, pw
        outs.append(out)
    _check(_load().bs_bitserial_conv2d_nhwc_tcw_group(ctypes.cast(descs, ctypes.c_void_p), len(convs), a_bits, w_bits,
                                                      _stream(stream)))
    return outs
