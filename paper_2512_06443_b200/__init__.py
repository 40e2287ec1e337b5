"""paper_2512_06443_b200 -- B200-native Vec-LUT ternary mpGeMM (arXiv 2512.06443).

Thin Python binding over the C ABI of ``libvlut.so`` (``include/vlut.h``):
argument marshalling only.  Every step of the hot path (table build, lookup,
accumulation, split-K reduction, dequant, quantization, packing on device)
runs in the CUDA kernels of ``csrc/``; PyTorch is used only for device memory,
streams and ``torch.distributed``.  There is no CPU fallback: if the library
is missing or no CUDA device is present, calls raise.

The binding keeps the C names: ``packed_bytes``, ``pack_weights``,
``pack_weights_device``, ``mpgemm``, ``mpgemm_ex``, ``mpgemm_acc``,
``quantize``, ``plan``, ``last_error``.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

__all__ = [
    "VlutError", "PackedWeights", "LaunchPlan", "lib", "lib_path", "packed_bytes",
    "pack_weights", "pack_weights_device", "unpack_weights_host", "plan", "mpgemm",
    "mpgemm_ex", "mpgemm_acc", "quantize", "last_error", "EXPORTS", "group_schedule",
    "mpgemm_decode",
    "MixedPackedWeights", "pack_weights_mixed", "mpgemm_mixed", "mpgemm_layout", "quantize_t",
    "linear", "workspace", "plan_ws", "mpgemm_ws", "mpgemm_acc_ws", "mpgemm_fused",
    "quantize_amax", "mpgemm_scalar_lut", "slot_plan", "mpgemm_allgather",
    "cached_workspaces", "release_workspaces",
]

_HERE = os.path.dirname(os.path.abspath(__file__))
lib_path = os.path.join(_HERE, "libvlut.so")

STATUS = {
    0: "VLUT_OK", 1: "VLUT_ERR_INVALID_ARGUMENT", 2: "VLUT_ERR_INVALID_TRIT",
    3: "VLUT_ERR_SHAPE", 4: "VLUT_ERR_BUFFER_TOO_SMALL", 5: "VLUT_ERR_MISALIGNED",
    6: "VLUT_ERR_CORRUPT_DESCRIPTOR", 7: "VLUT_ERR_CUDA", 8: "VLUT_ERR_UNSUPPORTED",
}
VLUT_MAGIC = 0x31544C56
VLUT_VERSION = 1


class VlutError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.name = STATUS.get(status, str(status))


class _Desc(ctypes.Structure):
    _fields_ = [
        ("magic", ctypes.c_uint32), ("version", ctypes.c_uint32),
        ("M", ctypes.c_int32), ("K", ctypes.c_int32), ("g", ctypes.c_int32),
        ("m_pad", ctypes.c_int32), ("kg_tiles", ctypes.c_int32),
        ("m_tile", ctypes.c_int32), ("kg_tile", ctypes.c_int32),
        ("flags", ctypes.c_int32), ("payload_bytes", ctypes.c_int64),
        ("payload", ctypes.c_void_p),
    ]


class _Plan(ctypes.Structure):
    _fields_ = [("warps", ctypes.c_int32), ("splits", ctypes.c_int32),
                ("m_cta", ctypes.c_int32), ("n_cta", ctypes.c_int32),
                ("grid_ctas", ctypes.c_int32), ("smem_bytes", ctypes.c_int32),
                ("streamk", ctypes.c_int32), ("slot", ctypes.c_int32),
                ("tpw", ctypes.c_int32), ("nw", ctypes.c_int32)]


# Every symbol include/vlut.h declares (tests check the .so exports them all).
EXPORTS = {
    "vlut_packed_bytes": ([ctypes.c_int, ctypes.c_int, ctypes.c_int], ctypes.c_size_t),
    "vlut_pack_weights": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                           ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(_Desc),
                           ctypes.c_void_p], ctypes.c_int),
    "vlut_pack_weights_device": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                  ctypes.c_void_p, ctypes.c_size_t, ctypes.POINTER(_Desc),
                                  ctypes.c_void_p], ctypes.c_int),
    "vlut_packed_bytes_ex": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int],
                             ctypes.c_size_t),
    "vlut_pack_weights_ex": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                              ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                              ctypes.POINTER(_Desc), ctypes.c_void_p], ctypes.c_int),
    "vlut_pack_weights_device_ex": ([ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                                     ctypes.POINTER(_Desc), ctypes.c_void_p], ctypes.c_int),
    "vlut_unpack_weights_host": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p],
                                 ctypes.c_int),
    "vlut_plan": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                   ctypes.POINTER(_Plan)], ctypes.c_int),
    "vlut_mpgemm": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_float,
                     ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                     ctypes.c_void_p], ctypes.c_int),
    "vlut_mpgemm_ex": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p,
                        ctypes.c_float, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                        ctypes.c_int, ctypes.POINTER(_Plan), ctypes.c_void_p], ctypes.c_int),
    "vlut_mpgemm_acc": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p,
                         ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Plan),
                         ctypes.c_void_p], ctypes.c_int),
    "vlut_quantize": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                       ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "vlut_quantize_ex": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                          ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p],
                         ctypes.c_int),
    "vlut_group_schedule": ([ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                             ctypes.POINTER(ctypes.c_int)], ctypes.c_int),
    "vlut_mpgemm_mixed": ([ctypes.POINTER(_Desc), ctypes.POINTER(_Desc), ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p, ctypes.c_int,
                           ctypes.c_int, ctypes.c_int, ctypes.c_void_p], ctypes.c_int),
    "vlut_mpgemm_layout": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p,
                            ctypes.c_float, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                            ctypes.c_int, ctypes.c_int, ctypes.c_void_p], ctypes.c_int),
    "vlut_quantize_t": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "vlut_linear": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p,
                     ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                     ctypes.c_void_p], ctypes.c_int),
    "vlut_workspace_bytes": ([], ctypes.c_size_t),
    "vlut_mpgemm_ws": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p, ctypes.c_float,
                        ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                        ctypes.POINTER(_Plan), ctypes.c_void_p, ctypes.c_size_t,
                        ctypes.c_void_p], ctypes.c_int),
    "vlut_mpgemm_acc_ws": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p,
                            ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_Plan),
                            ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p], ctypes.c_int),
    "vlut_plan_ws": ([ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                      ctypes.POINTER(_Plan)], ctypes.c_int),
    "vlut_mpgemm_mixed_ws": ([ctypes.POINTER(_Desc), ctypes.POINTER(_Desc), ctypes.c_void_p,
                              ctypes.c_void_p, ctypes.c_float, ctypes.c_void_p, ctypes.c_int,
                              ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
                              ctypes.c_void_p], ctypes.c_int),
    "vlut_mpgemm_fused": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_float, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                           ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int,
                           ctypes.POINTER(_Plan), ctypes.c_void_p, ctypes.c_size_t,
                           ctypes.c_void_p], ctypes.c_int),
    "vlut_quantize_amax": ([ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p], ctypes.c_int),
    "vlut_mpgemm_scalar_lut": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p,
                                ctypes.c_float, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                ctypes.c_int, ctypes.POINTER(_Plan), ctypes.c_void_p,
                                ctypes.c_size_t, ctypes.c_void_p], ctypes.c_int),
    "vlut_mpgemm_decode": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_float,
                            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                            ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p], ctypes.c_int),
    "vlut_mpgemm_allgather": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p,
                               ctypes.c_float, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                               ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                               ctypes.c_int, ctypes.c_void_p], ctypes.c_int),
    "vlut_mpgemm_allgather_multicast": ([ctypes.POINTER(_Desc), ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.c_float, ctypes.c_void_p, ctypes.c_int,
                                         ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.c_void_p], ctypes.c_int),
    "vlut_launches_per_mpgemm": ([], ctypes.c_int),
    "vlut_cached_workspaces": ([], ctypes.c_int),
    "vlut_release_workspaces": ([], ctypes.c_int),
    "vlut_active_clusters": ([ctypes.c_int, ctypes.c_int, ctypes.c_int], ctypes.c_int),
    "vlut_last_error": ([], ctypes.c_char_p),
    "vlut_version": ([], ctypes.c_char_p),
}

_lib = None


def lib() -> ctypes.CDLL:
    """Load libvlut.so (built in-tree by ``__graft_entry__.build()``).  Raises
    if it is missing -- there is deliberately no fallback."""
    global _lib
    if _lib is None:
        if not os.path.exists(lib_path):
            raise RuntimeError(f"{lib_path} is missing: run `python -c 'import __graft_entry__ "
                               f"as g; g.build()'` (there is no CPU fallback)")
        L = ctypes.CDLL(lib_path)
        for name, (args, res) in EXPORTS.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def last_error() -> str:
    return lib().vlut_last_error().decode()


def _check(st: int) -> None:
    if st != 0:
        raise VlutError(st, last_error())


def _stream(stream, device=None):
    """The stream to launch on: ``stream``, else the current stream of
    ``device`` (the device of the call's tensors), never another GPU's."""
    import torch
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return stream


def _stream_ptr(stream, device=None) -> ctypes.c_void_p:
    return ctypes.c_void_p(_stream(stream, device).cuda_stream)


def _dev_ptr(t) -> ctypes.c_void_p:
    if t is None:
        return ctypes.c_void_p(0)
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _arg(t, name: str, dtype, shape=None, device=None, optional: bool = False):
    """Device pointer of tensor ``t`` after checking what the C entry point
    will assume about it (dtype, exact shape, device, contiguity): a wrong
    dtype or a short buffer would otherwise be read or written past its end."""
    import torch
    if t is None:
        if optional:
            return ctypes.c_void_p(0)
        raise ValueError(f"{name}: required")
    if not isinstance(t, torch.Tensor):
        raise TypeError(f"{name}: expected a torch tensor")
    if not t.is_cuda:
        raise ValueError(f"{name}: expected a CUDA tensor (no CPU fallback)")
    if t.dtype != dtype:
        raise TypeError(f"{name}: expected {dtype}, got {t.dtype}")
    if shape is not None and tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: expected shape {tuple(shape)}, got {tuple(t.shape)}")
    if device is not None and t.device != device:
        raise ValueError(f"{name}: on {t.device}, expected {device}")
    if not t.is_contiguous():
        raise ValueError(f"{name}: expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _act(A):
    """(K, N, device) of int8 activations [K][N]."""
    import torch
    if not isinstance(A, torch.Tensor) or A.dim() != 2:
        raise ValueError("A: expected a 2-D int8 CUDA tensor [K][N]")
    if A.dtype != torch.int8:
        raise TypeError(f"A: expected torch.int8, got {A.dtype}")
    return int(A.shape[0]), int(A.shape[1]), A.device


def _ws_arg(ws, device):
    import torch
    if ws is None:
        return ctypes.c_void_p(0), 0
    return _arg(ws, "ws", torch.uint8, device=device), int(ws.numel())


@dataclass
class LaunchPlan:
    warps: int
    splits: int = 1
    m_cta: int = 0
    n_cta: int = 64
    grid_ctas: int = 0
    smem_bytes: int = 0
    streamk: int = 0
    slot: int = 0   # 1: K2 lane-slot kernel (small N / decode / scalar-LUT comparator)
    tpw: int = 0    # K2 tokens per table word: 1 = scalar LUT (1->1), 2 = vector (1->2)
    nw: int = 0     # K2 table words per lookup (0 = heuristic)

    def _c(self) -> _Plan:
        return _Plan(self.warps, self.splits, self.m_cta, self.n_cta, self.grid_ctas,
                     self.smem_bytes, self.streamk, self.slot, self.tpw, self.nw)

    @staticmethod
    def _from_c(p: "_Plan") -> "LaunchPlan":
        return LaunchPlan(p.warps, p.splits, p.m_cta, p.n_cta, p.grid_ctas, p.smem_bytes,
                          p.streamk, p.slot, p.tpw, p.nw)


def slot_plan(tpw: int = 2, nw: int = 0, splits: int = 0) -> LaunchPlan:
    """A K2 plan: tpw 1 (scalar LUT) or 2 (vector); nw / splits 0 = heuristic."""
    return LaunchPlan(warps=16, splits=splits, n_cta=0, slot=1, tpw=tpw, nw=nw)


class PackedWeights:
    """Device payload tensor + the C descriptor (a1)."""

    def __init__(self, payload, desc: _Desc):
        self.payload = payload  # keeps the device memory alive
        self.desc = desc

    @property
    def M(self):
        return self.desc.M

    @property
    def K(self):
        return self.desc.K

    @property
    def g(self):
        return self.desc.g

    @property
    def nbytes(self):
        return int(self.desc.payload_bytes)


PACK_PAD_K = 1  # VLUT_PACK_PAD_K: K need not be a multiple of g (zero-trit padding)


def packed_bytes(M: int, K: int, g: int, flags: int = 0) -> int:
    return int(lib().vlut_packed_bytes_ex(M, K, g, flags))


def pack_weights(w_trits: np.ndarray, g: int, device=None, stream=None,
                 pad_k: bool = False) -> PackedWeights:
    """Host trits int8 [M][K] -> device packed weights (validated on host).
    pad_k: allow K % g != 0 (the last group is completed with zero trits)."""
    import torch
    w = np.ascontiguousarray(w_trits, dtype=np.int8)
    M, K = w.shape
    flags = PACK_PAD_K if pad_k else 0
    nb = packed_bytes(M, K, g, flags)
    if nb == 0:
        raise VlutError(3, f"cannot pack M={M} K={K} g={g}")
    payload = torch.empty(nb, dtype=torch.uint8, device=device or "cuda")
    d = _Desc()
    with torch.cuda.device(payload.device):
        _check(lib().vlut_pack_weights_ex(ctypes.c_void_p(w.ctypes.data), M, K, g, flags,
                                          _dev_ptr(payload), nb, ctypes.byref(d),
                                          _stream_ptr(stream, payload.device)))
    return PackedWeights(payload, d)


def pack_weights_device(w_trits, g: int, stream=None, pad_k: bool = False) -> PackedWeights:
    """Device trits (torch int8 CUDA [M][K]) -> packed weights, on the GPU."""
    import torch
    if w_trits.dim() != 2:
        raise ValueError("w_trits: expected [M][K]")
    M, K = w_trits.shape
    flags = PACK_PAD_K if pad_k else 0
    nb = packed_bytes(M, K, g, flags)
    if nb == 0:
        raise VlutError(3, f"cannot pack M={M} K={K} g={g}")
    payload = torch.empty(nb, dtype=torch.uint8, device=w_trits.device)
    d = _Desc()
    with torch.cuda.device(payload.device):
        _check(lib().vlut_pack_weights_device_ex(_arg(w_trits, "w_trits", torch.int8),
                                                 M, K, g, flags,
                                                 _dev_ptr(payload), nb, ctypes.byref(d),
                                                 _stream_ptr(stream, payload.device)))
    return PackedWeights(payload, d)


def unpack_weights_host(pw: PackedWeights) -> np.ndarray:
    host = pw.payload.cpu().numpy()
    out = np.zeros((pw.M, pw.K), dtype=np.int8)
    _check(lib().vlut_unpack_weights_host(ctypes.byref(pw.desc),
                                          ctypes.c_void_p(host.ctypes.data),
                                          ctypes.c_void_p(out.ctypes.data)))
    return out


def plan(M: int, K: int, N: int, g: int) -> LaunchPlan:
    p = _Plan()
    _check(lib().vlut_plan(M, K, N, g, ctypes.byref(p)))
    return LaunchPlan._from_c(p)


def _plan_ptr(p: Optional[LaunchPlan]):
    if p is None:
        return None, ctypes.POINTER(_Plan)()
    c = p._c()
    return c, ctypes.byref(c)


def _weights(W: PackedWeights, K: int, dev):
    if W.K != K:
        raise ValueError(f"W has K={W.K}, A has {K} rows")
    if W.payload.device != dev:
        raise ValueError(f"W payload on {W.payload.device}, A on {dev}")
    return ctypes.byref(W.desc)


def _out(out, shape, dtype, dev, name="out"):
    import torch
    if out is None:
        out = torch.empty(shape, dtype=dtype, device=dev)
    return out, _arg(out, name, dtype, shape, dev)


def mpgemm_ex(W: PackedWeights, A, a_scale, w_scale: float, out=None,
              plan: Optional[LaunchPlan] = None, stream=None):
    """fp32 out[M][N] = dequant(W x A) (a2-a6).  A: torch int8 CUDA [K][N]."""
    import torch
    K, N, dev = _act(A)
    M = W.M
    out, op = _out(out, (M, N), torch.float32, dev)
    keep, pp = _plan_ptr(plan)
    with torch.cuda.device(dev):
        _check(lib().vlut_mpgemm_ex(_weights(W, K, dev), _dev_ptr(A),
                                    _arg(a_scale, "a_scale", torch.float32, (N,), dev),
                                    float(w_scale), op, M, K, N, pp, _stream_ptr(stream, dev)))
    return out


def mpgemm(W: PackedWeights, A, a_scale, w_scale: float, out=None, stream=None):
    """The north-star entry point vlut_mpgemm(W_packed, A_int8, a_scale,
    w_scale, out, M, K, N, stream)."""
    import torch
    K, N, dev = _act(A)
    M = W.M
    out, op = _out(out, (M, N), torch.float32, dev)
    with torch.cuda.device(dev):
        _check(lib().vlut_mpgemm(_weights(W, K, dev), _dev_ptr(A),
                                 _arg(a_scale, "a_scale", torch.float32, (N,), dev),
                                 float(w_scale), op, M, K, N, _stream_ptr(stream, dev)))
    return out


def mpgemm_acc(W: PackedWeights, A, out=None, plan: Optional[LaunchPlan] = None, stream=None):
    """Raw int32 accumulators [M][N] (bit-exact test hook)."""
    import torch
    K, N, dev = _act(A)
    M = W.M
    out, op = _out(out, (M, N), torch.int32, dev)
    keep, pp = _plan_ptr(plan)
    with torch.cuda.device(dev):
        _check(lib().vlut_mpgemm_acc(_weights(W, K, dev), _dev_ptr(A), op, M, K, N, pp,
                                     _stream_ptr(stream, dev)))
    return out


def quantize(x, y=None, q=None, scale=None, stream=None, cluster: int = 0):
    """Per-token absmax int8 quantizer of fp32 [K][N] (x * y if y given).
    cluster: K3 CTAs per 16-token block (0 = the library's choice; 1 for a
    quantizer overlapping an mpGeMM on another stream, see vlut_quantize_ex)."""
    import torch
    if x.dim() != 2:
        raise ValueError("x: expected fp32 [K][N]")
    K, N = x.shape
    dev = x.device
    q, qp = _out(q, (K, N), torch.int8, dev, "q")
    scale, sp = _out(scale, (N,), torch.float32, dev, "scale")
    with torch.cuda.device(dev):
        _check(lib().vlut_quantize_ex(_arg(x, "x", torch.float32, device=dev),
                                      _arg(y, "y", torch.float32, (K, N), dev, optional=True),
                                      K, N, qp, sp, int(cluster), _stream_ptr(stream, dev)))
    return q, scale


# ---------------------------------------------------------------- mixed g=5/g=4 (f2)
def group_schedule(K: int):
    """(k5, k4): features packed with g=5 first, then g=4."""
    k5, k4 = ctypes.c_int(0), ctypes.c_int(0)
    _check(lib().vlut_group_schedule(K, ctypes.byref(k5), ctypes.byref(k4)))
    return k5.value, k4.value


class MixedPackedWeights:
    """A (g=5 part, g=4 part) pair covering K = k5 + k4 (either may be None)."""

    def __init__(self, w5: Optional[PackedWeights], w4: Optional[PackedWeights], M: int, K: int):
        self.w5, self.w4, self.M, self.K = w5, w4, M, K

    @property
    def nbytes(self):
        return sum(w.nbytes for w in (self.w5, self.w4) if w is not None)


def pack_weights_mixed(w_trits: np.ndarray, device=None, stream=None) -> MixedPackedWeights:
    """Host trits int8 [M][K] -> the mixed g=5/g=4 packing (~1.6 BPW for any
    representable K)."""
    w = np.ascontiguousarray(w_trits, dtype=np.int8)
    M, K = w.shape
    k5, k4 = group_schedule(K)
    w5 = pack_weights(np.ascontiguousarray(w[:, :k5]), 5, device, stream) if k5 else None
    w4 = pack_weights(np.ascontiguousarray(w[:, k5:]), 4, device, stream) if k4 else None
    return MixedPackedWeights(w5, w4, M, K)


def mpgemm_mixed(W: MixedPackedWeights, A, a_scale, w_scale: float, out=None, ws=None,
                 stream=None):
    import torch
    K, N, dev = _act(A)
    if W.K != K:
        raise ValueError(f"W has K={W.K}, A has {K} rows")
    out, op = _out(out, (W.M, N), torch.float32, dev)
    d5 = ctypes.byref(W.w5.desc) if W.w5 is not None else ctypes.POINTER(_Desc)()
    d4 = ctypes.byref(W.w4.desc) if W.w4 is not None else ctypes.POINTER(_Desc)()
    wsp, wsn = _ws_arg(ws, dev)
    with torch.cuda.device(dev):
        _check(lib().vlut_mpgemm_mixed_ws(d5, d4, _dev_ptr(A),
                                          _arg(a_scale, "a_scale", torch.float32, (N,), dev),
                                          float(w_scale), op, W.M, K, N, wsp, wsn,
                                          _stream_ptr(stream, dev)))
    return out


# ---------------------------------------------------------------- feature-major layouts (f3)
OUT_FEATURE_MAJOR = 1


def mpgemm_layout(W: PackedWeights, A, a_scale, w_scale: float, out=None, feature_major=True,
                  stream=None):
    """vlut_mpgemm with the fused output transposition: out [N][M] if feature_major."""
    import torch
    K, N, dev = _act(A)
    M = W.M
    out, op = _out(out, (N, M) if feature_major else (M, N), torch.float32, dev)
    with torch.cuda.device(dev):
        _check(lib().vlut_mpgemm_layout(_weights(W, K, dev), _dev_ptr(A),
                                        _arg(a_scale, "a_scale", torch.float32, (N,), dev),
                                        float(w_scale), op, M, K, N,
                                        OUT_FEATURE_MAJOR if feature_major else 0,
                                        _stream_ptr(stream, dev)))
    return out


def quantize_t(x_nk, y_nk=None, q=None, scale=None, stream=None):
    """Per-token quantizer of feature-major fp32 [N][K] -> (int8 [K][N], fp32 [N])."""
    import torch
    if x_nk.dim() != 2:
        raise ValueError("x_nk: expected fp32 [N][K]")
    N, K = x_nk.shape
    dev = x_nk.device
    q, qp = _out(q, (K, N), torch.int8, dev, "q")
    scale, sp = _out(scale, (N,), torch.float32, dev, "scale")
    with torch.cuda.device(dev):
        _check(lib().vlut_quantize_t(_arg(x_nk, "x_nk", torch.float32, device=dev),
                                     _arg(y_nk, "y_nk", torch.float32, (N, K), dev, optional=True),
                                     K, N, qp, sp, _stream_ptr(stream, dev)))
    return q, scale


def linear(W: PackedWeights, x_nk, w_scale: float, y=None, q_ws=None, s_ws=None, stream=None):
    """Framework-layout ternary linear: x fp32 [N][K] -> y fp32 [N][M]."""
    import torch
    if x_nk.dim() != 2:
        raise ValueError("x_nk: expected fp32 [N][K]")
    N, K = x_nk.shape
    dev = x_nk.device
    y, yp = _out(y, (N, W.M), torch.float32, dev, "y")
    q_ws, qp = _out(q_ws, (K, N), torch.int8, dev, "q_ws")
    s_ws, sp = _out(s_ws, (N,), torch.float32, dev, "s_ws")
    with torch.cuda.device(dev):
        _check(lib().vlut_linear(_weights(W, K, dev), _arg(x_nk, "x_nk", torch.float32, device=dev),
                                 float(w_scale), yp, W.M, K, N, qp, sp, _stream_ptr(stream, dev)))
    return y


# ---------------------------------------------------------------- workspaces
# One workspace per (device, stream): a workspace is used by one stream at a
# time (vlut.h), and calls on one stream are ordered.  Bounded: a fifth stream
# on a device evicts the least recently used entry after synchronising the
# device (the evicted entry's stream may still be using it).
_WS = {}
_WS_CAP = 4
_ws_tick = 0


def workspace(device=None, stream=None):
    """The zeroed workspace of (device, stream) (stream None: that device's
    current stream) for the *_ws entry points."""
    import torch
    global _ws_tick
    dev = torch.device(device or "cuda")
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    st = _stream(stream, dev)
    key = (dev.index, int(st.cuda_stream))
    _ws_tick += 1
    ent = _WS.get(key)
    if ent is not None:
        ent[1] = _ws_tick
        return ent[0]
    same = [k for k in _WS if k[0] == dev.index]
    with torch.cuda.device(dev):
        if len(same) >= _WS_CAP:
            torch.cuda.synchronize(dev)
            del _WS[min(same, key=lambda k: _WS[k][1])]
        nb = int(lib().vlut_workspace_bytes())
        if nb == 0:
            raise VlutError(7, "no CUDA device for the stream-K workspace")
        with torch.cuda.stream(st):
            ws = torch.zeros(nb, dtype=torch.uint8, device=dev)
    _WS[key] = [ws, _ws_tick]
    return ws


def cached_workspaces() -> int:
    """Workspaces the C library keeps for vlut_mpgemm (all devices)."""
    return int(lib().vlut_cached_workspaces())


def release_workspaces() -> None:
    """Free the C library's vlut_mpgemm workspaces and this module's."""
    import torch
    _check(lib().vlut_release_workspaces())
    if _WS:
        for d in {k[0] for k in _WS}:
            torch.cuda.synchronize(d)
        _WS.clear()


def plan_ws(M: int, K: int, N: int, g: int) -> LaunchPlan:
    p = _Plan()
    _check(lib().vlut_plan_ws(M, K, N, g, ctypes.byref(p)))
    return LaunchPlan._from_c(p)


def mpgemm_ws(W: PackedWeights, A, a_scale, w_scale: float, out=None,
              plan: Optional[LaunchPlan] = None, ws=None, stream=None):
    """vlut_mpgemm with a workspace: the planner may pick the stream-K schedule.
    ws None: the workspace of (A's device, the launch stream)."""
    import torch
    K, N, dev = _act(A)
    M = W.M
    st = _stream(stream, dev)
    out, op = _out(out, (M, N), torch.float32, dev)
    if ws is None:
        ws = workspace(dev, st)
    wsp, wsn = _ws_arg(ws, dev)
    keep, pp = _plan_ptr(plan)
    with torch.cuda.device(dev):
        _check(lib().vlut_mpgemm_ws(_weights(W, K, dev), _dev_ptr(A),
                                    _arg(a_scale, "a_scale", torch.float32, (N,), dev),
                                    float(w_scale), op, M, K, N, pp, wsp, wsn,
                                    ctypes.c_void_p(st.cuda_stream)))
    return out


def mpgemm_acc_ws(W: PackedWeights, A, out=None, plan: Optional[LaunchPlan] = None, ws=None,
                  stream=None):
    import torch
    K, N, dev = _act(A)
    M = W.M
    st = _stream(stream, dev)
    out, op = _out(out, (M, N), torch.int32, dev)
    if ws is None:
        ws = workspace(dev, st)
    wsp, wsn = _ws_arg(ws, dev)
    keep, pp = _plan_ptr(plan)
    with torch.cuda.device(dev):
        _check(lib().vlut_mpgemm_acc_ws(_weights(W, K, dev), _dev_ptr(A), op, M, K, N,
                                        pp, wsp, wsn, ctypes.c_void_p(st.cuda_stream)))
    return out


# ---------------------------------------------------------------- fused re-quantization (f1)
def mpgemm_fused(W: PackedWeights, A, a_scale, w_scale: float, out=None, mul_in=None,
                 amax=None, amax_rows: Optional[int] = None,
                 plan: Optional[LaunchPlan] = None, ws=None, stream=None):
    """mpGeMM whose epilogue multiplies by mul_in ([M][N] fp32, optional) and
    atomically maxes |out| over rows < amax_rows into amax (int32 [N] viewed
    as float bits; zero it first).  Returns out."""
    import torch
    K, N, dev = _act(A)
    M = W.M
    out, op = _out(out, (M, N), torch.float32, dev)
    rows = M if amax_rows is None else amax_rows
    wsp, wsn = _ws_arg(ws, dev)
    keep, pp = _plan_ptr(plan)
    with torch.cuda.device(dev):
        _check(lib().vlut_mpgemm_fused(_weights(W, K, dev), _dev_ptr(A),
                                       _arg(a_scale, "a_scale", torch.float32, (N,), dev),
                                       float(w_scale), op, M, K, N,
                                       _arg(mul_in, "mul_in", torch.float32, (M, N), dev,
                                            optional=True),
                                       _arg(amax, "amax", torch.int32, (N,), dev, optional=True),
                                       int(rows), pp, wsp, wsn, _stream_ptr(stream, dev)))
    return out


def quantize_amax(x, amax, q=None, scale=None, stream=None):
    """Quantize fp32 [K][N] with per-token maxima already known (f1)."""
    import torch
    if x.dim() != 2:
        raise ValueError("x: expected fp32 [K][N]")
    K, N = x.shape
    dev = x.device
    q, qp = _out(q, (K, N), torch.int8, dev, "q")
    scale, sp = _out(scale, (N,), torch.float32, dev, "scale")
    with torch.cuda.device(dev):
        _check(lib().vlut_quantize_amax(_arg(x, "x", torch.float32, device=dev),
                                        _arg(amax, "amax", torch.int32, (N,), dev),
                                        K, N, qp, sp, _stream_ptr(stream, dev)))
    return q, scale


# ---------------------------------------------------------------- scalar-LUT comparator (f4)
def mpgemm_scalar_lut(W: PackedWeights, A, a_scale, w_scale: float, out=None,
                      plan: Optional[LaunchPlan] = None, ws=None, use_ws: bool = True,
                      stream=None):
    """The scalar-LUT (1->1, one table per token) mpGeMM on the K2 kernel
    (P:84-85); with use_ws the K range is split across CTAs."""
    import torch
    K, N, dev = _act(A)
    M = W.M
    st = _stream(stream, dev)
    out, op = _out(out, (M, N), torch.float32, dev)
    if ws is None and use_ws:
        ws = workspace(dev, st)
    wsp, wsn = _ws_arg(ws, dev)
    keep, pp = _plan_ptr(plan)
    with torch.cuda.device(dev):
        _check(lib().vlut_mpgemm_scalar_lut(_weights(W, K, dev), _dev_ptr(A),
                                            _arg(a_scale, "a_scale", torch.float32, (N,), dev),
                                            float(w_scale), op, M, K, N, pp, wsp, wsn,
                                            ctypes.c_void_p(st.cuda_stream)))
    return out


def mpgemm_decode(W: PackedWeights, x, w_scale: float, out=None, scale_out=None, ws=None,
                  stream=None):
    """Fused decode step (N = 1): fp32 activations x [K] (or [K][1]) -> fp32
    out [M], quantization inside the K2 decode kernel (vlut_mpgemm_decode);
    bit-identical to quantize() + mpgemm_scalar_lut().  Returns (out, scale)."""
    import torch
    if x.dim() == 2 and x.shape[1] == 1:
        x = x.reshape(-1)
    if x.dim() != 1:
        raise ValueError("x: expected fp32 [K] (one token)")
    K = x.shape[0]
    dev = x.device
    M = W.M
    st = _stream(stream, dev)
    xp = _arg(x, "x", torch.float32, (K,), dev)
    out, op = _out(out, (M,), torch.float32, dev)
    scale_out, sp = _out(scale_out, (1,), torch.float32, dev, "scale_out")
    if ws is None:
        ws = workspace(dev, st)
    wsp, wsn = _ws_arg(ws, dev)
    with torch.cuda.device(dev):
        _check(lib().vlut_mpgemm_decode(_weights(W, K, dev), xp, float(w_scale), op, sp, M, K,
                                        wsp, wsn, ctypes.c_void_p(st.cuda_stream)))
    return out, scale_out


# ---------------------------------------------------------------- fused all-gather (a8)
def mpgemm_allgather(W: PackedWeights, A, a_scale, w_scale: float, out_full, row0: int,
                     peer_ptrs=(), stream=None, multicast: bool = False):
    """Shard rows [row0, row0 + W.M) of out_full [M_total][N] (a tensor or a
    raw device address), stored there and to every peer buffer in
    ``peer_ptrs`` (device pointers mapped into this process) by the K1
    epilogue.  multicast=True: out_full is a multicast address (an int; no
    peers) and the epilogue stores through it with multimem.st.  Returns
    out_full."""
    import torch
    K, N, dev = _act(A)
    if multicast:
        if not isinstance(out_full, int) or peer_ptrs:
            raise ValueError("multicast: out_full must be the multicast address, no peers")
        with torch.cuda.device(dev):
            _check(lib().vlut_mpgemm_allgather_multicast(
                _weights(W, K, dev), _dev_ptr(A), _arg(a_scale, "a_scale", torch.float32, (N,), dev),
                float(w_scale), ctypes.c_void_p(out_full), W.M, K, N, int(row0),
                _stream_ptr(stream, dev)))
        return out_full
    arr = (ctypes.c_void_p * max(1, len(peer_ptrs)))(*[ctypes.c_void_p(int(x)) for x in peer_ptrs])
    # out_full: a tensor, or a raw device address (e.g. a multicast address)
    if isinstance(out_full, int):
        out_p = ctypes.c_void_p(int(out_full))
    else:
        if out_full.dim() != 2 or out_full.shape[1] != N or out_full.shape[0] < row0 + W.M:
            raise ValueError("out_full: expected fp32 [>= row0 + M][N]")
        out_p = _arg(out_full, "out_full", torch.float32, device=dev)
    with torch.cuda.device(dev):
        _check(lib().vlut_mpgemm_allgather(_weights(W, K, dev), _dev_ptr(A),
                                           _arg(a_scale, "a_scale", torch.float32, (N,), dev),
                                           float(w_scale), out_p, W.M, K, N, int(row0),
                                           ctypes.cast(arr, ctypes.POINTER(ctypes.c_void_p)),
                                           len(peer_ptrs), _stream_ptr(stream, dev)))
    return out_full
