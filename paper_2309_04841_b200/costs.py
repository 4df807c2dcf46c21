"""Device-resident cost diagonals (float64 and lossless uint16 levels).

The reference keeps one host float64 vector per problem (qaoa.py:71-87).
Here a ``DeviceCosts`` owns the GPU copy of that vector (bit-identical to the
reference's) and, when the diagonal lies on a 16-bit grid (every LABS /
MaxCut / integer-weight instance), a uint16 level vector in the
``CompactCostVector`` encoding (terms.py:123-175) — 2 B instead of 8 B per
amplitude streamed by the phase and expectation passes.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .terms import TermPolynomial, _infer_n, precompute_device, term_arrays


class DeviceCosts:
    """Cost diagonal of one (shard of a) problem on the current CUDA device."""

    def __init__(self, n: int, f64: torch.Tensor | None = None, u16: torch.Tensor | None = None,
                 scale: float = 1.0, offset: float = 0.0, levels: int = 0):
        self.n = n
        self.levels = int(levels)  # uint16: 1 + largest level (sizes the phase tables); 0 = unknown
        self.f64 = f64
        self.u16 = u16
        self.scale = float(scale)
        self.offset = float(offset)
        self._minmax: tuple[float, float] | None = None
        self._host: np.ndarray | None = None

    # -------------------------------------------------------------- constructors
    @classmethod
    def from_polynomial(cls, poly: TermPolynomial, compact: bool = True, keep_f64: bool = True,
                        index_base: int = 0, n_local: int | None = None) -> "DeviceCosts":
        n_local = poly.n if n_local is None else n_local
        size = 1 << n_local
        if keep_f64:
            dc = cls(n_local, f64=precompute_device(poly, index_base, size))
            if compact:
                dc.try_compact()
            return dc
        # uint16 only: exact-integer levels straight from the terms (no float64 vector)
        dc = cls(n_local)
        if not dc._levels_from_terms(poly, index_base, size):
            raise MemoryError("cost diagonal is not on a 16-bit grid and the float64 vector was not kept")
        return dc

    @classmethod
    def from_array(cls, costs, compact: bool = True) -> "DeviceCosts":
        dev = _lib.device()
        if isinstance(costs, torch.Tensor):
            t = costs.to(device=dev, dtype=torch.float64).contiguous()
        else:
            arr = np.ascontiguousarray(costs, dtype=np.float64)
            if not arr.flags.writeable:  # e.g. the reference's read-only memoised diagonal (qaoa.py:74)
                arr = arr.copy()
            t = torch.from_numpy(arr).to(dev)
        n = _infer_n(t.numel())  # the reference's error for malformed lengths (terms.py:178-182)
        dc = cls(n, f64=t)
        if compact:
            dc.try_compact()
        return dc

    # -------------------------------------------------------------- encodings
    def try_compact(self) -> bool:
        """Pack into uint16 levels if lossless (device-checked bit-for-bit)."""
        if self.f64 is None:
            return self.u16 is not None
        lo, hi = self.minmax()
        if not (np.isfinite(lo) and np.isfinite(hi)):
            return False
        for scale in self._candidate_scales():
            if (hi - lo) / scale > 65535.0:
                continue
            u16 = torch.empty(self.f64.numel(), dtype=torch.uint16, device=self.f64.device)
            bad = torch.zeros(1, dtype=torch.int32, device=self.f64.device)
            _lib.call("fq_compact_u16", u16.data_ptr(), self.f64.data_ptr(), self.f64.numel(), scale, lo,
                      bad.data_ptr(), _lib.stream())
            if int(bad.item()) == 0:
                self.u16, self.scale, self.offset = u16, scale, lo
                self.levels = int(round((hi - lo) / scale)) + 1
                return True
        return False

    def _candidate_scales(self):
        yield 1.0
        for s in range(1, 8):
            yield 2.0 ** -s

    def _levels_from_terms(self, poly: TermPolynomial, index_base: int, size: int) -> bool:
        ta = term_arrays(poly)
        if ta.iweights is None:
            return False
        dev = _lib.device()
        iw = torch.from_numpy(ta.iweights).to(dev)
        m = torch.from_numpy(ta.masks).to(dev)
        acc_bits = 32 if ta.abs_sum < 2 ** 31 else 64
        # level offset: the global minimum is unknown without a pass; use the
        # lower bound -sum|w| then shift to the observed minimum is not needed
        # for correctness (decode uses the same offset).  Range check: sum|w|*2 levels.
        lo = -ta.abs_sum
        if 2 * ta.abs_sum > 65535:
            return False
        out = torch.empty(size, dtype=torch.uint16, device=dev)
        bad = torch.zeros(1, dtype=torch.int32, device=dev)
        chunk = min(size, 1 << 28)
        if size >= 4096 and index_base % chunk == 0:
            # Walsh-Hadamard transform per 2^28-amplitude chunk into a float64 scratch
            # (2 GiB), then lossless packing: no float64 vector of the whole shard
            tmp = torch.empty(chunk, dtype=torch.float64, device=dev)
            scale, offset = 2.0 ** -ta.shift, float(lo) * 2.0 ** -ta.shift
            for c0 in range(0, size, chunk):
                _lib.call("fq_precompute_wht", tmp.data_ptr(), chunk, iw.data_ptr(), m.data_ptr(), len(poly.terms),
                          ta.shift, index_base + c0, _lib.stream())
                _lib.call("fq_compact_u16", out[c0:c0 + chunk].data_ptr(), tmp.data_ptr(), chunk, scale, offset,
                          bad.data_ptr(), _lib.stream())
            del tmp
        else:
            _lib.call("fq_precompute_levels_u16", out.data_ptr(), size, iw.data_ptr(), m.data_ptr(),
                      len(poly.terms), acc_bits, index_base, lo, 0, bad.data_ptr(), _lib.stream())
        if int(bad.item()) != 0:
            return False
        self.u16 = out
        self.scale = 2.0 ** -ta.shift
        self.offset = float(lo) * self.scale
        # the levels were packed from the bound -sum|w|: move the origin to the
        # observed minimum (exact: dyadic values) so the phase tables (levels <
        # 16384) cover the range in use, e.g. LABS n = 34 (2 sum|w| + 1 > 16384)
        c_lo, c_hi = self.minmax()
        delta = int(round((c_lo - self.offset) / self.scale))
        _lib.call("fq_rebase_u16", out.data_ptr(), size, delta, _lib.stream())
        self.offset += delta * self.scale
        self.levels = int(round((c_hi - c_lo) / self.scale)) + 1
        return True

    # -------------------------------------------------------------- views
    @property
    def size(self) -> int:
        return 1 << self.n

    def kernel_view(self):
        """(cost_kind, pointer, scale, offset) the fused kernels stream."""
        if self.u16 is not None:
            return _lib.COST_U16, self.u16.data_ptr(), self.scale, self.offset
        return _lib.COST_F64, self.f64.data_ptr(), 1.0, 0.0

    def minmax(self) -> tuple[float, float]:
        if self._minmax is None:
            out = torch.empty(2, dtype=torch.float64, device=_lib.device())
            kind, p, scale, offset = self.kernel_view() if self.f64 is None else (_lib.COST_F64, self.f64.data_ptr(), 1.0, 0.0)
            _lib.call("fq_cost_minmax", p, kind, scale, offset, self.size, out.data_ptr(),
                      _lib.scratch().data_ptr(), _lib.stream())
            lo, hi = out.tolist()
            self._minmax = (lo, hi)
        return self._minmax

    def host(self) -> np.ndarray:
        """Host float64 copy (read-only), like the reference's cached vector."""
        if self._host is None:
            if self.f64 is not None:
                arr = self.f64.cpu().numpy()
            else:
                arr = self.scale * self.u16.cpu().numpy().astype(np.float64) + self.offset
            arr.setflags(write=False)
            self._host = arr
        return self._host

    def nbytes_per_amp(self) -> int:
        return 2 if self.u16 is not None else 8
