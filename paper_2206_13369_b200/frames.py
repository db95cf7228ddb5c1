"""Frame-stack pipeline (reference io.py:131-182, cli.py:311-334 ``video``)
on the B200 solvers.

PGM parsing and file writes stay on the host (they are file I/O).  The
layout work runs on the device: only the 8-bit rasters cross PCIe (1 byte per
pixel each way, not 8), ``frames_to_matrix`` builds the solver matrix in HBM
(pixel (row, col) of frame j -> entry (row + col*H, j), scaled by 1/255) and
``matrix_to_frames`` quantizes L and S back to 8-bit frames (clamp to [0, 1],
round half up), so ingest -> emit reproduces the input bytes exactly, as the
reference promises (io.py:161-166).
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .api_types import CpcpOptions, PcpOptions
from .runtime import require_cuda


class FormatError(ValueError):
    """Input bytes do not conform to the expected file format (io.py:28-29)."""


@dataclass
class FrameStack:
    """io.py:32-43: one frame per column; ``matrix`` is a numpy array, or a
    CUDA tensor when ingested with ``device_matrix=True``."""

    frame_height: int
    frame_width: int
    count: int
    matrix: object


_PGM_SPACE = frozenset(b" \t\n\r\x0b\x0c")


def _pgm_header(buf, path):
    """Scan the P5 header of an in-memory PGM file.

    Returns (width, height, maxval, raster offset).  Header fields are
    whitespace-separated decimal tokens; '#' opens a comment that runs to the
    end of the line and may appear anywhere in the header; the raster starts
    right after the single whitespace byte that ends the maxval field
    (the header grammar of reference io.py:83-114)."""
    if buf[:2] != b"P5":
        raise FormatError(f"{path}: not a binary PGM (P5) file")
    pos, n, fields = 2, len(buf), []
    while len(fields) < 3:
        digits = bytearray()
        while True:
            if pos >= n:
                raise FormatError("unexpected end of PGM header")
            c = buf[pos]
            pos += 1
            if c == 0x23:  # '#': drop the rest of the line
                nl = buf.find(b"\n", pos)
                pos = n if nl < 0 else nl + 1
            elif c in _PGM_SPACE:
                if digits:
                    break
            else:
                digits.append(c)
        fields.append(int(bytes(digits)))
    width, height, maxval = fields
    return width, height, maxval, pos


def read_pgm(path):
    """Binary 8-bit PGM (P5) -> (height, width) uint8 (reference io.py:100-114)."""
    with open(path, "rb") as fh:
        buf = fh.read()
    width, height, maxval, off = _pgm_header(buf, path)
    if maxval != 255:
        raise FormatError(f"{path}: only 8-bit PGM supported, maxval={maxval}")
    count = width * height
    if len(buf) - off < count:
        raise FormatError(f"{path}: truncated raster")
    return np.frombuffer(buf, dtype=np.uint8, count=count, offset=off).reshape((height, width)).copy()


def write_pgm(pixels, path):
    """(height, width) uint8 -> canonical binary PGM: 'P5\\n<w> <h>\\n255\\n'
    then the raster (reference io.py:117-125)."""
    img = np.asarray(pixels, dtype=np.uint8)
    if img.ndim != 2:
        raise ValueError("pixels must be 2-D")
    header = b"P5\n%d %d\n255\n" % (img.shape[1], img.shape[0])
    with open(path, "wb") as fh:
        fh.write(header + np.ascontiguousarray(img).tobytes())


def read_frames(paths):
    """All frames as one (count, height, width) uint8 array, validated like
    ingest_frames (io.py:134-147)."""
    paths = list(paths)
    if not paths:
        raise ValueError("no frames given")
    first = read_pgm(paths[0])
    height, width = first.shape
    out = np.empty((len(paths), height, width), dtype=np.uint8)
    out[0] = first
    for j, path in enumerate(paths[1:], start=1):
        frame = read_pgm(path)
        if frame.shape != (height, width):
            raise ValueError(f"{path}: frame is {frame.shape[0]}x{frame.shape[1]}, expected {height}x{width}")
        out[j] = frame
    return out


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def frames_to_matrix(raster, dtype=torch.float64, device=None):
    """(count, H, W) uint8 (numpy or torch) -> (H*W) x count device matrix."""
    require_cuda()
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    r = raster if isinstance(raster, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(raster))
    if r.dtype != torch.uint8 or r.dim() != 3:
        raise ValueError("raster must be a (count, height, width) uint8 array")
    if not r.is_cuda:
        r = r.pin_memory().to(dev, non_blocking=True)
    r = r.contiguous()
    count, h, w = r.shape
    x = torch.empty((h * w, count), dtype=dtype, device=dev)
    with torch.cuda.device(dev):
        _lib.check(_lib.load().mlr_frames_to_matrix(ctypes.c_void_p(r.data_ptr()), count, h, w,
                                                    int(dtype == torch.float32), ctypes.c_void_p(x.data_ptr()),
                                                    x.stride(0), _stream()))
    return x


def matrix_to_frames(x, height, width):
    """(H*W) x count matrix (numpy or torch) -> (count, H, W) uint8 numpy,
    quantized on the device (io.py:153-158)."""
    require_cuda()
    t = x if isinstance(x, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(x))
    if t.dtype not in (torch.float32, torch.float64):
        t = t.to(torch.float64)
    if not t.is_cuda:
        t = t.to(torch.device("cuda", torch.cuda.current_device()))
    t = t.contiguous()
    m, count = t.shape
    if m != height * width:
        raise ValueError("component shapes do not match the frame stack")
    out = torch.empty((count, height, width), dtype=torch.uint8, device=t.device)
    with torch.cuda.device(t.device):
        _lib.check(_lib.load().mlr_matrix_to_frames(ctypes.c_void_p(t.data_ptr()), t.stride(0),
                                                    int(t.dtype == torch.float32), count, height, width,
                                                    ctypes.c_void_p(out.data_ptr()), _stream()))
    return out.cpu().numpy()


def ingest_frames(paths, dtype=np.float64, device_matrix=False):
    """Drop-in for io.ingest_frames (io.py:128-150): PGM frames -> FrameStack
    with pixel values scaled to [0, 1].  The matrix is built on the GPU;
    ``device_matrix=True`` leaves it there (a CUDA tensor) for the solvers."""
    raster = read_frames(paths)
    tdt = torch.float32 if np.dtype(dtype) == np.float32 else torch.float64
    x = frames_to_matrix(raster, tdt)
    count, h, w = raster.shape
    return FrameStack(frame_height=h, frame_width=w, count=count, matrix=x if device_matrix else x.cpu().numpy())


def emit_frames(stack, l, s, out_dir):
    """Drop-in for io.emit_frames (io.py:161-182): l_XXXX.pgm / s_XXXX.pgm per
    frame; returns the written paths in the reference's order."""
    shape = tuple(stack.matrix.shape)
    if tuple(l.shape) != shape or tuple(s.shape) != shape:
        raise ValueError("component shapes do not match the frame stack")
    fl = matrix_to_frames(l, stack.frame_height, stack.frame_width)
    fs = matrix_to_frames(s, stack.frame_height, stack.frame_width)
    os.makedirs(out_dir, exist_ok=True)
    digits = max(4, len(str(stack.count - 1)))
    written = []
    for j in range(stack.count):
        for tag, frames in (("l", fl), ("s", fs)):
            path = os.path.join(out_dir, f"{tag}_{j:0{digits}d}.pgm")
            write_pgm(frames[j], path)
            written.append(path)
    return written


def video(paths, out_dir=None, solver="ml-fwt", opts=None, dtype=np.float64):
    """The reference's ``video`` command (cli.py:311-334) on the GPU: ingest,
    solve with the matrix resident in HBM, emit L/S frames.  ``opts`` defaults
    to the CLI's (cli.py:179-207: lambda_l = 1/sqrt(max(m, n)), lambda_s =
    lambda_l/sqrt(max(m, n)), tol 1e-3, 2000 iterations for the CPCP solvers;
    tol 1e-7, 500 iterations for PCP).  Returns (state, stack, written paths)."""
    from .cpcp import fwt_solve, ml_fwt_solve
    from .pcp import ialm_solve, ml_ialm_solve
    stack = ingest_frames(paths, dtype, device_matrix=True)
    d = stack.matrix
    if solver in ("ml-fwt", "fwt"):
        if opts is None:
            big = max(d.shape)
            lam_l = 1.0 / np.sqrt(big)
            opts = CpcpOptions(lambda_l=lam_l, lambda_s=lam_l / np.sqrt(big), tol=1e-3, max_iters=2000,
                               collect_rank=False)
        state = (ml_fwt_solve if solver == "ml-fwt" else fwt_solve)(d, None, opts)
    elif solver in ("ml-ialm", "ialm"):
        opts = opts if opts is not None else PcpOptions()
        state = (ml_ialm_solve if solver == "ml-ialm" else ialm_solve)(d, opts)
    else:
        raise ValueError(f"unknown solver {solver!r}")
    written = emit_frames(stack, state.l, state.s, out_dir) if out_dir is not None else []
    return state, stack, written
