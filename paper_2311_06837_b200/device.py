"""Device-side data layout and thin wrappers over the libgdx kernels.

PyTorch is used only as the device allocator / stream provider: tensors are
raw HBM buffers whose pointers are handed to the C ABI.  Layout rules:

* CSR: row_ptr int64[rows+1] (u64 offsets), col int32[nnz] (u32 ids);
* fp32 dense matrices: row pitch padded to a multiple of 4 (16-byte rows);
* split-bf16 GEMM operands: hi/lo int16 arrays, row pitch padded to a
  multiple of 8 (16-byte TMA pitch), zero-filled padding.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import AggregateArgs, GemmArgs, call, ptr
from .errors import InputError, InternalError


def pad4(x: int) -> int:
    return (x + 3) // 4 * 4


def pad8(x: int) -> int:
    return (x + 7) // 8 * 8


def require_cuda():
    if not torch.cuda.is_available():
        raise InternalError("no CUDA device visible: the B200 engine has no CPU fallback")


def stream_handle(stream=None) -> int:
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


@dataclass
class DeviceCSR:
    row_ptr: torch.Tensor  # int64 [rows+1]
    col: torch.Tensor      # int32 [nnz]
    rows: int

    @staticmethod
    def upload(ro: np.ndarray, ci: np.ndarray, device) -> "DeviceCSR":
        require_cuda()
        rp = torch.from_numpy(np.ascontiguousarray(ro).view(np.int64)).to(device, non_blocking=False)
        c = torch.from_numpy(np.ascontiguousarray(ci).view(np.int32) if len(ci) else
                             np.zeros(1, np.int32)).to(device)
        return DeviceCSR(rp, c, len(ro) - 1)

    def slice_rows(self, lo: int, hi: int) -> "DeviceCSR":
        """Rows [lo, hi): offsets stay absolute into the same col array."""
        return DeviceCSR(self.row_ptr[lo:hi + 1], self.col, hi - lo)

    @property
    def nnz(self) -> int:
        return int(self.row_ptr[-1].item() - self.row_ptr[0].item())


class Split:
    """Split-bf16 matrix (x = hi + lo) with rows x cols logical shape, pitch ld."""

    def __init__(self, rows: int, cols: int, device, ld: int | None = None):
        self.rows, self.cols = rows, cols
        self.ld = pad8(cols) if ld is None else ld
        self.hi = torch.zeros(max(rows, 1) * self.ld, dtype=torch.int16, device=device)
        self.lo = torch.zeros(max(rows, 1) * self.ld, dtype=torch.int16, device=device)

    def rows_view(self, rows: int) -> "Split":
        """The first `rows` rows (same storage)."""
        v = Split.__new__(Split)
        v.rows, v.cols, v.ld, v.hi, v.lo = rows, self.cols, self.ld, self.hi, self.lo
        return v

    def to_float(self) -> torch.Tensor:
        """fp32 value (for tests): hi + lo."""
        def f(t):
            return (t.view(self.rows if self.rows else 1, self.ld)[:self.rows, :self.cols]
                    .to(torch.int32).bitwise_left_shift(16).view(torch.float32))
        return f(self.hi) + f(self.lo)

    def fill_from(self, x: torch.Tensor, ld_x: int, transpose: bool = False, stream=None):
        """hi/lo := split(x) (x: fp32, logical rows x cols if not transpose, else cols x rows)."""
        if transpose:
            call("gdx_split_bf16", x.data_ptr(), ld_x, self.cols, self.rows, self.hi.data_ptr(),
                 self.lo.data_ptr(), self.ld, 1, stream_handle(stream))
        else:
            call("gdx_split_bf16", x.data_ptr(), ld_x, self.rows, self.cols, self.hi.data_ptr(),
                 self.lo.data_ptr(), self.ld, 0, stream_handle(stream))
        return self


def dense(rows: int, cols: int, device, zero: bool = True) -> torch.Tensor:
    """fp32 matrix storage with a 16-byte row pitch; returns a [rows, pad4(cols)] tensor."""
    f = torch.zeros if zero else torch.empty
    return f((max(rows, 1), pad4(cols)), dtype=torch.float32, device=device)


def aggregate(g: DeviceCSR, src: torch.Tensor, width: int, *, out=None, out_split: Split | None = None,
              self_coef: float = 0.0, self_base: int = 0, post_scale=None, add=None, relu=False,
              row_end=None, row_begin=None, skip=None, partial=None, stream=None, variant: int = 0,
              bins: "RowBins | None" = None, src_lo8=None, ld_src_lo8: int = 0):
    """K1/K3 (see include/gdx.h gdx_aggregate).  row_begin/row_end override the CSR
    row bounds; skip = (seg_lo, seg_hi) excludes a per-row sub-range; partial adds
    precomputed partial sums before the epilogue.  src_lo8 (uint8 tensor or byte
    address): src is the u16 high plane of packed-24 rows, this the low plane (pitch
    ld_src_lo8 bytes, default the high plane's pitch in elements)."""
    a = AggregateArgs()
    a.row_ptr = g.row_ptr.data_ptr() if row_begin is None else row_begin.data_ptr()
    a.row_end = ptr(row_end) if row_begin is None else (row_end.data_ptr() if row_end is not None
                                                         else g.row_ptr[1:].data_ptr())
    if skip is not None:
        a.skip_lo, a.skip_hi = skip[0].data_ptr(), skip[1].data_ptr()
    if partial is not None:
        a.partial, a.ld_partial = partial.data_ptr(), partial.stride(0)
    a.col = g.col.data_ptr()
    a.rows = g.rows
    a.width = width
    a.src = src.data_ptr()
    a.ld_src = src.stride(0) if src.dim() == 2 else width
    if src_lo8 is not None:
        a.src_lo8 = src_lo8 if isinstance(src_lo8, int) else src_lo8.data_ptr()
        a.ld_src_lo8 = ld_src_lo8
    a.self_coef = self_coef
    a.self_base = self_base
    a.post_scale = ptr(post_scale)
    a.add = ptr(add)
    a.ld_add = add.stride(0) if add is not None else 0
    a.relu = int(relu)
    a.out = ptr(out)
    a.ld_out = out.stride(0) if out is not None else 0
    if out_split is not None:
        a.out_hi, a.out_lo, a.ld_split = out_split.hi.data_ptr(), out_split.lo.data_ptr(), out_split.ld
    if bins is not None:
        call("gdx_aggregate_balanced", _lib.C.byref(a), variant, bins._p, stream_handle(stream))
    elif variant:
        call("gdx_aggregate_variant", _lib.C.byref(a), variant, stream_handle(stream))
    else:
        call("gdx_aggregate", _lib.C.byref(a), stream_handle(stream))


class RowBins:
    """Degree bins of a CSR (gdx_row_bins_build): rows above heavy_degree are split into
    chunk_edges-edge chunks; pass as aggregate(..., bins=) for skewed graphs."""

    def __init__(self, row_ptr_host: np.ndarray, heavy_degree: int, chunk_edges: int = 1024,
                 max_width: int = 256):
        rp = np.ascontiguousarray(row_ptr_host, np.uint64)
        self._p = _lib.C.POINTER(_lib.RowBins)()
        call("gdx_row_bins_build", rp.ctypes.data, len(rp) - 1, heavy_degree, chunk_edges, max_width,
             _lib.C.byref(self._p))
        b = self._p.contents
        self.n_light, self.n_heavy, self.n_chunks = b.n_light, b.n_heavy, b.n_chunks

    def __del__(self):
        try:
            if self._p:
                _lib.lib().gdx_row_bins_free(self._p)
        except Exception:
            pass


def gemm_tn(A: Split, B: Split, *, c0=None, c1=None, split=None, row_scale=None, relu=False,
            out_split: Split | None = None, split_k: int = 1, m=None, simt=False, a_mn=False,
            b_mn=False, mask=None, split_unscaled=False, peers=None, stream=None, a_rows=None,
            b_rows=None, p24=None):
    """K2: C(m, n) = sum_k A(m, k) B(n, k).  A is stored [m][k] (K-major) or, with
    a_mn, [k][m]; likewise B ([n][k] or [k][n]).  a_rows / b_rows (int32 device
    tensors): A / B are the SOURCE matrices and the operand's rows (m for a K-major A,
    k for an MN-major B) are gathered through the index.  See gdx_gemm_tn."""
    mA, kA = (A.cols, A.rows) if a_mn else (A.rows, A.cols)
    nB, kB = (B.cols, B.rows) if b_mn else (B.rows, B.cols)
    if a_rows is not None:
        mA = a_rows.numel()
    if b_rows is not None:
        kB = b_rows.numel()
    assert kA == kB, (kA, kB)
    g = GemmArgs()
    g.a_hi, g.a_lo, g.lda = A.hi.data_ptr(), A.lo.data_ptr(), A.ld
    g.b_hi, g.b_lo, g.ldb = B.hi.data_ptr(), B.lo.data_ptr(), B.ld
    g.a_mn_major, g.b_mn_major = int(a_mn), int(b_mn)
    g.m = mA if m is None else m
    g.n = nB
    g.k = kA
    for c in (c0, c1):
        if c is not None and (c.dim() != 2 or c.stride(1) != 1):
            raise InputError("gemm_tn: outputs must be 2-D row-major views (unit column stride)")
    g.c0 = ptr(c0)
    g.ldc0 = c0.stride(0) if c0 is not None else 0
    g.c1 = ptr(c1)
    g.ldc1 = c1.stride(0) if c1 is not None else 0
    g.split = nB if split is None else split
    g.row_scale = ptr(row_scale)
    g.relu = int(relu)
    if out_split is not None:
        g.out_hi, g.out_lo, g.ld_split = out_split.hi.data_ptr(), out_split.lo.data_ptr(), out_split.ld
    g.split_k = split_k
    if mask is not None:
        g.mask, g.ld_mask = mask.data_ptr(), mask.stride(0)
    g.split_unscaled = int(split_unscaled)
    if p24 is not None:   # (hi address, lo address, ld_hi u16, ld_lo bytes, target output)
        g.p24_hi, g.p24_lo, g.ld_p24_hi, g.ld_p24_lo, g.p24_target = p24
    if a_rows is not None:
        g.a_rows, g.a_src_rows = a_rows.data_ptr(), A.rows
    if b_rows is not None:
        g.b_rows, g.b_src_rows = b_rows.data_ptr(), B.rows
    if peers is not None:  # (target output, byte deltas): fused NVLink exchange
        target, deltas = peers
        g.npeers, g.peer_target = len(deltas), int(target)
        for i, dl in enumerate(deltas):
            g.peer_delta[i] = int(dl)
    call("gdx_gemm_tn_simt" if simt else "gdx_gemm_tn", _lib.C.byref(g), stream_handle(stream))


def degree_scale(g: DeviceCSR, kind: int, device) -> torch.Tensor:
    out = torch.empty(max(g.rows, 1), dtype=torch.float32, device=device)
    call("gdx_degree_scale", g.row_ptr.data_ptr(), g.rows, kind, out.data_ptr(), stream_handle())
    return out
