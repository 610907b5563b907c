"""Dequantization after decode on the GPU.

Mirrors the reference's reconstruction API (quant.py:25-74): ``QuantConfig``
(error bound, symbol width -> midpoint), ``QuantResult`` (codes plus the
outlier sidecar) and ``dequantize`` (kernels.py:216-227 ``dequantize_chain``:
``pred = f64(f32(pred + 2eb * (code - midpoint)))``, outliers reset ``pred``
to their stored value).  The quantizer itself is out of scope.

On the device (csrc/quant.cu):

* exact regime -- 2eb a power of two and every outlier value a multiple of
  it: one pass, a segmented prefix sum with a decoupled look-back, writing the
  float64 reconstruction at HBM speed.  The kernel flags any running sum that
  leaves +-2^24 (where float32 rounding would start to lose bits);
* otherwise, or when the flag is raised: the reference recurrence itself on
  one device thread -- bit-identical in every regime, but sequential.

``decode_dequantize`` runs decode and reconstruction back to back on the
device, so the uint16 codes never leave it.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from ._lib import check, load, ptr, require_cuda, stream_handle
from .device import h2d


@dataclass(frozen=True)
class QuantConfig:
    """quant.py:25-36."""

    error_bound: float
    symbol_width: int = 16

    def __post_init__(self):
        if not self.error_bound > 0:
            raise ValueError(f"error bound must be > 0, got {self.error_bound}")
        if self.symbol_width not in (8, 16):
            raise ValueError(f"symbol width must be 8 or 16, got {self.symbol_width}")

    @property
    def midpoint(self) -> int:
        return 1 << (self.symbol_width - 1)


@dataclass
class QuantResult:
    """quant.py:39-47."""

    codes: np.ndarray
    outlier_indices: np.ndarray
    outlier_values: np.ndarray

    @property
    def outliers(self) -> list[tuple[int, float]]:
        return list(zip(self.outlier_indices.tolist(), self.outlier_values.tolist()))


def exact_regime(twice_eb: float, outlier_values) -> tuple[bool, np.ndarray]:
    """Whether the one-pass scan may run: 2eb = 2^e (-149 <= e <= 104) and each
    outlier value an integer multiple of 2eb below 2^24 of them.  Returns the
    outlier values in units of 2eb."""
    m, e = np.frexp(twice_eb)
    if m != 0.5 or not (-149 <= e - 1 <= 104):
        return False, np.zeros(0, np.int64)
    v = np.asarray(outlier_values, dtype=np.float64)
    u = v / twice_eb  # exact: division by a power of two
    ok = bool(np.all(np.isfinite(u)) and np.all(np.abs(u) < 2.0 ** 24) and np.all(u == np.rint(u)))
    return ok, (np.rint(u).astype(np.int64) if ok else np.zeros(0, np.int64))


def dequantize_device(codes_dev, n: int, outlier_indices, outlier_values, config: QuantConfig,
                      stats: dict | None = None):
    """float64 reconstruction (device tensor) of n uint16 codes on the device."""
    torch = require_cuda()
    lib = load()
    dev = codes_dev.device
    twice_eb = 2.0 * float(config.error_bound)
    mid = config.midpoint
    oi = np.ascontiguousarray(outlier_indices, dtype=np.int64)
    ov = np.ascontiguousarray(outlier_values, dtype=np.float64)
    if oi.size != ov.size:
        raise ValueError("outlier indices and values differ in length")
    if oi.size > 1 and np.any(np.diff(oi) <= 0):
        raise ValueError("outlier indices must be strictly increasing")
    out = torch.empty(max(n, 1), dtype=torch.float64, device=dev)
    src = codes_dev if codes_dev.data_ptr() % 16 == 0 else codes_dev.clone()
    oi_d = h2d(oi if oi.size else np.zeros(1, np.int64), dev)
    exact, units = exact_regime(twice_eb, ov)
    path = "chain"
    if exact:
        u_d = h2d(units if units.size else np.zeros(1, np.int64), dev)
        wsb = lib.bh_dequant_workspace_bytes(n)
        ws = torch.empty(wsb, dtype=torch.uint8, device=dev)
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
        check(lib.bh_dequantize(ptr(src), n, ptr(oi_d), None, ptr(u_d), oi.size, twice_eb, mid, 1, ptr(out),
                                ptr(ws), wsb, ptr(flag), stream_handle()), "dequantize")
        if int(flag.item()) == 0:
            path = "scan"
    if path == "chain":
        ov_d = h2d(ov if ov.size else np.zeros(1, np.float64), dev)
        check(lib.bh_dequantize(ptr(src), n, ptr(oi_d), ptr(ov_d), None, oi.size, twice_eb, mid, 0, ptr(out),
                                None, 0, None, stream_handle()), "dequantize")
    if stats is not None:
        stats["path"] = path
    return out[:n]


def dequantize(result: QuantResult, config: QuantConfig) -> np.ndarray:
    """quant.py:64-74 on the device: float64 reconstruction of the codes."""
    torch = require_cuda()
    codes = np.ascontiguousarray(result.codes, dtype=np.uint16)
    dev = torch.device("cuda", torch.cuda.current_device())
    cd = h2d(codes if codes.size else np.zeros(1, np.uint16), dev)
    out = dequantize_device(cd, codes.size, result.outlier_indices, result.outlier_values, config)
    return out.cpu().numpy()[: codes.size]


def decode_dequantize(stream, outlier_indices, outlier_values, config: QuantConfig, variant: str = "gap",
                      device_out: bool = False, stats: dict | None = None):
    """Decode a stream and reconstruct its values on the device (the codes stay there)."""
    from . import gap_decoder, sync_decoder
    dec = gap_decoder if variant == "gap" else sync_decoder
    codes = dec.decode(stream, device_out=True)
    out = dequantize_device(codes, int(stream.symbol_count), outlier_indices, outlier_values, config, stats)
    return out if device_out else out.cpu().numpy()
