"""Range compression into device-resident complex64 envelopes.

Mirrors rangecomp.range_compress (/root/reference/pkg/src/hhsar/rangecomp.py:
61-101): an unnormalised zero-padded inverse DFT over the n_f frequency
samples to n_t = upsample * n_f delay bins, then demodulation from the band
start to the band-centre carrier k_ref.  For power-of-two n_t in [16, 8192]
(every BASELINE config) this is one fused kernel (hhsar_range_compress:
pad + radix-16 Stockham IDFT + demodulation in a single HBM pass, or
hhsar_range_compress_window for a delay-bin window); other n_t, or
HHSAR_RANGE_FFT=cufft, use a batched cuFFT through torch.fft (norm="forward"
= no 1/n factor) followed by the hhsar_range_demod kernel (float64 phase per
bin).  The result stays in HBM
as envelopes[N_el][n_t] complex64, time fastest -- the layout every
backprojection kernel reads.
"""

from __future__ import annotations

import os
import threading
import warnings
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ConfigError
from .model import C_LIGHT


@dataclass(frozen=True)
class RangeProfileSet:
    """RangeProfileSet (rangecomp.py:24-58) with device envelopes.

    ``envelopes`` is a CUDA complex64 tensor [N_el, n_t]; ``elements_dev`` the
    float64 element positions on the same device.
    """

    envelopes: object
    t0: float
    dt: float
    upsample: int
    k_ref: float
    aperture: object
    freqs: object
    elements_dev: object = None

    @property
    def n_samples(self) -> int:
        return int(self.envelopes.shape[1])

    @property
    def window(self) -> tuple:
        return (self.t0, self.t0 + (self.n_samples - 1) * self.dt)


# The fused single-pass kernel (hhsar_range_compress: register radix-16
# Stockham passes, pad + IDFT + demodulation in one HBM pass) agrees with the
# cuFFT path to 2e-7 and is 2x faster on B200 (config 3: 1.13 vs 2.28 ms);
# HHSAR_RANGE_FFT=cufft selects the cuFFT + hhsar_range_demod path.
_FORCE_CUFFT = os.environ.get("HHSAR_RANGE_FFT", "fused") == "cufft"


def profile_axis(freqs, upsample: int):
    """(n_t, dt, k_ref, a) exactly as rangecomp.py:84-96 computes them;
    a = (k_min - k_ref) * c is the demodulation rate per second of delay."""
    if int(upsample) != upsample or upsample < 1:
        raise ConfigError("upsample factor must be an integer >= 1")
    upsample = int(upsample)
    k_min, k_max = freqs.k_min, freqs.k_max
    dk = (k_max - k_min) / (freqs.count - 1)
    n_t = upsample * freqs.count
    dt = 2.0 * np.pi / (n_t * dk * C_LIGHT)
    k_ref = 0.5 * (k_min + k_max)
    return n_t, dt, k_ref, (k_min - k_ref) * C_LIGHT


def _host_tensor(values):
    import torch
    if isinstance(values, torch.Tensor):
        return values
    arr = np.ascontiguousarray(values, dtype=np.complex64)
    with warnings.catch_warnings():  # read-only (frozen) arrays are only read here
        warnings.simplefilter("ignore", UserWarning)
        return torch.from_numpy(arr)


def to_device_cube(values, device="cuda", stream=None):
    """Host complex cube -> device complex64 (one copy; see upload_cube for
    the chunked, overlappable form)."""
    import torch
    if isinstance(values, torch.Tensor):
        return values.to(device=device, dtype=torch.complex64, non_blocking=True)
    host = _host_tensor(values)
    if not host.is_pinned():
        # staging copy: pageable host memory cannot be DMA'd asynchronously
        return host.to(device)
    return host.to(device, non_blocking=True)


_LOCAL = threading.local()  # per host thread: copy streams, pinned staging buffers
UPLOAD_CHUNK_BYTES = 256 << 20


def _local(name):
    d = getattr(_LOCAL, name, None)
    if d is None:
        d = {}
        setattr(_LOCAL, name, d)
    return d


def copy_stream(device):
    """Per-device (and per host thread) stream for host->device uploads."""
    import torch
    streams = _local("streams")
    key = torch.device(device).index
    if key not in streams:
        streams[key] = torch.cuda.Stream(device=device)
    return streams[key]


class CubeUpload:
    """A cube on its way to the device: ``tensor`` (complex64 [rows, n_f] in
    HBM) is filled chunk by chunk on a copy stream; ``chunks`` lists (r0, r1,
    event) with the event recorded once rows [r0, r1) have landed, so
    consumers (range compression) can start on early chunks while later
    ones are still crossing PCIe.  Pinned host input is DMA'd directly
    (every chunk queued at once); pageable input goes through two reused
    pinned staging buffers (host copy of chunk i+1 overlaps the DMA of
    chunk i)."""

    def __init__(self, values, device="cuda", rows=None, chunk_bytes: int | None = None):
        import torch
        dev = torch.device(device)
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        host = _host_tensor(values)
        r0, r1 = rows if rows is not None else (0, host.shape[0])
        n_f = host.shape[1]
        self.row0 = r0
        self.tensor = torch.empty((r1 - r0, n_f), dtype=torch.complex64, device=dev)
        self.chunks = []
        self.h2d_bytes = (r1 - r0) * n_f * 8
        if r1 == r0:
            return
        step = max(1, int((chunk_bytes or UPLOAD_CHUNK_BYTES) // (n_f * 8)))
        cs = copy_stream(dev)
        cs.wait_stream(torch.cuda.current_stream(dev))  # the destination is allocated
        pinned = host.is_pinned() and host.dtype == torch.complex64
        if pinned:
            with torch.cuda.stream(cs):
                for a in range(r0, r1, step):
                    b = min(r1, a + step)
                    self.tensor[a - r0:b - r0].copy_(host[a:b], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                    self.chunks.append((a, b, ev))
        else:
            staging = _local("staging")
            bufs = staging.get((dev.index, step, n_f))
            if bufs is None:
                bufs = [(torch.empty((step, n_f), dtype=torch.complex64, pin_memory=True),
                         torch.cuda.Event()) for _ in range(2)]
                staging.clear()
                staging[(dev.index, step, n_f)] = bufs
            src = host.numpy() if host.device.type == "cpu" else None
            for i, a in enumerate(range(r0, r1, step)):
                b = min(r1, a + step)
                buf, free = bufs[i % 2]
                free.synchronize()  # its previous DMA has finished
                if src is not None:
                    np.copyto(buf[:b - a].numpy(), src[a:b], casting="same_kind")
                else:
                    buf[:b - a].copy_(host[a:b])
                with torch.cuda.stream(cs):
                    self.tensor[a - r0:b - r0].copy_(buf[:b - a], non_blocking=True)
                    ev = torch.cuda.Event()
                    ev.record(cs)
                free.record(cs)
                self.chunks.append((a, b, ev))
        self.tensor.record_stream(cs)

    def wait(self, stream=None):
        """Make ``stream`` (default: current) wait for every chunk."""
        import torch
        s = stream or torch.cuda.current_stream()
        for _, _, ev in self.chunks:
            s.wait_event(ev)


def range_compress_device(cube_dev, freqs, upsample: int = 8):
    """Device cube [N_el, n_f] complex64 -> envelopes [N_el, n_t] complex64."""
    import torch
    n_t, dt, k_ref, a = profile_axis(freqs, upsample)
    if cube_dev.dtype != torch.complex64:
        cube_dev = cube_dev.to(torch.complex64)
    if 16 <= n_t <= 8192 and n_t & (n_t - 1) == 0 and not _FORCE_CUFFT:
        # one fused pass: pad + IDFT + demodulation (hhsar_range_compress)
        cube_dev = cube_dev.contiguous()
        prof = torch.empty((cube_dev.shape[0], n_t), dtype=torch.complex64,
                           device=cube_dev.device)
        _native.call("hhsar_range_compress", _native.ptr(cube_dev), cube_dev.shape[0],
                     cube_dev.shape[1], n_t, a, dt, _native.ptr(prof), _native.stream_handle())
        return prof, dt, k_ref
    prof = torch.fft.ifft(cube_dev, n=n_t, dim=1, norm="forward")
    if prof.dtype != torch.complex64:
        prof = prof.to(torch.complex64)
    prof = prof.contiguous()
    _native.call("hhsar_range_demod", _native.ptr(prof), prof.shape[0], n_t, a, dt, 1.0,
                 _native.stream_handle())
    return prof, dt, k_ref


def range_compress_window(cube_dev, freqs, upsample: int, b0: int, w: int, out=None,
                          chunks=None, row0: int = 0):
    """Device cube -> the delay-bin window [b0, b0 + w) of every envelope row
    (hhsar_range_compress_window).  Returns (envelopes [N_el, w], t0', dt,
    k_ref): the gated rows are profiles starting at t0' = b0 dt.

    ``chunks`` (a CubeUpload's (r0, r1, event) list, rows counted from
    ``row0``) compresses chunk by chunk, each launch waiting only for its
    own rows to land, so the compression overlaps the rest of the upload."""
    import torch
    n_t, dt, k_ref, a = profile_axis(freqs, upsample)
    if not (16 <= n_t <= 8192 and n_t & (n_t - 1) == 0):
        if chunks:
            for *_, ev in chunks:
                torch.cuda.current_stream().wait_event(ev)
        env, dt, k_ref = range_compress_device(cube_dev, freqs, upsample)
        return env[:, b0:b0 + w].contiguous(), b0 * dt, dt, k_ref
    if cube_dev.dtype != torch.complex64:
        cube_dev = cube_dev.to(torch.complex64)
    cube_dev = cube_dev.contiguous()
    if out is None:
        out = torch.empty((cube_dev.shape[0], w), dtype=torch.complex64, device=cube_dev.device)
    stream = torch.cuda.current_stream()
    parts = [(r0 - row0, r1 - row0, ev) for r0, r1, ev in chunks] if chunks else \
        [(0, cube_dev.shape[0], None)]
    for r0, r1, ev in parts:
        if ev is not None:
            stream.wait_event(ev)
        if r1 <= r0:
            continue
        _native.call("hhsar_range_compress_window", _native.c_void_p_offset(cube_dev, r0 * cube_dev.shape[1]),
                     r1 - r0, cube_dev.shape[1], n_t, a, dt, int(b0), int(w),
                     _native.c_void_p_offset(out, r0 * w), _native.stream_handle())
    return out, b0 * dt, dt, k_ref


def range_compress(cube, upsample: int = 8, device="cuda") -> RangeProfileSet:
    """range_compress (rangecomp.py:61-101) on the GPU."""
    import torch
    _native.library()
    n_t, dt, k_ref, _ = profile_axis(cube.freqs, upsample)
    cube_dev = to_device_cube(cube.values, device)
    env, dt, k_ref = range_compress_device(cube_dev, cube.freqs, upsample)
    el = torch.tensor(np.ascontiguousarray(cube.aperture.elements, dtype=np.float64),
                      device=device)
    return RangeProfileSet(envelopes=env, t0=0.0, dt=dt, upsample=int(upsample), k_ref=k_ref,
                           aperture=cube.aperture, freqs=cube.freqs, elements_dev=el)
