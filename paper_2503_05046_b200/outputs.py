"""Run artifacts from device state: MPRB v1 particle frames, CSV mirrors and
the contact wrench log (the reference's outputs.py).

Byte-compatible with the reference (outputs.py:3-15, 33-105): little-endian
``b"MPRB"``, u32 version 1, u32 flags (bit 0: velocities), u64 count, f64
time, then f64[n,3] positions (and velocities); text artifacts format floats
with ``%.17g``.

``AsyncFrameWriter`` keeps the writing off the critical path: it copies the
device tensors into pinned host buffers on a side stream (one D2H per frame,
ordered after the step's kernels by an event) and a background thread writes
the file, so the next coupling step overlaps the copy and the disk write.
"""

from __future__ import annotations

import queue
import struct
import threading
from pathlib import Path

import numpy as np
import torch

FRAME_MAGIC = b"MPRB"
FRAME_VERSION = 1


def _fmt(x: float) -> str:
    return f"{float(x):.17g}"


def frame_bytes(time: float, positions: np.ndarray, velocities: np.ndarray | None = None) -> bytes:
    pos = np.ascontiguousarray(positions, dtype="<f8")
    flags = 1 if velocities is not None else 0
    parts = [FRAME_MAGIC, struct.pack("<IIQd", FRAME_VERSION, flags, pos.shape[0], float(time)),
             pos.tobytes()]
    if velocities is not None:
        parts.append(np.ascontiguousarray(velocities, dtype="<f8").tobytes())
    return b"".join(parts)


def write_frame(path, time: float, positions, velocities=None) -> None:
    """Synchronous write (outputs.py:33-42); accepts device tensors or arrays."""
    def host(a):
        return a.detach().cpu().numpy() if isinstance(a, torch.Tensor) else np.asarray(a)
    Path(path).write_bytes(frame_bytes(time, host(positions),
                                       None if velocities is None else host(velocities)))


def read_frame(path):
    """(time, positions, velocities or None) (outputs.py:45-58)."""
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != FRAME_MAGIC:
            raise ValueError(f"{path}: not a frame file (magic {magic!r})")
        version, flags, count, time = struct.unpack("<IIQd", fh.read(24))
        if version != FRAME_VERSION:
            raise ValueError(f"{path}: unsupported frame version {version}")
        pos = np.frombuffer(fh.read(count * 24), dtype="<f8").reshape(count, 3)
        vel = np.frombuffer(fh.read(count * 24), dtype="<f8").reshape(count, 3) if flags & 1 else None
    return time, pos.copy(), None if vel is None else vel.copy()


def write_frame_csv(path, time: float, positions, velocities=None) -> None:
    """CSV mirror (outputs.py:61-72)."""
    pos = positions.detach().cpu().numpy() if isinstance(positions, torch.Tensor) else positions
    vel = velocities.detach().cpu().numpy() if isinstance(velocities, torch.Tensor) else velocities
    cols = ["x", "y", "z"] + (["vx", "vy", "vz"] if vel is not None else [])
    lines = [f"# time={_fmt(time)}", ",".join(cols)]
    for i in range(pos.shape[0]):
        row = [_fmt(a) for a in pos[i]]
        if vel is not None:
            row += [_fmt(a) for a in vel[i]]
        lines.append(",".join(row))
    Path(path).write_text("\n".join(lines) + "\n")


class ContactLogWriter:
    """CSV wrench log, one row per (step, logged body) (outputs.py:87-105)."""

    COLUMNS = ["time", "body", "fx", "fy", "fz", "tx", "ty", "tz"]

    def __init__(self, path, body_names: list[str]):
        self.body_names = list(body_names)
        self._fh = open(path, "w")
        self._fh.write(",".join(self.COLUMNS) + "\n")

    def log_step(self, time: float, wrench_rows: dict) -> None:
        for name in self.body_names:
            vals = ",".join(_fmt(v) for v in np.asarray(wrench_rows[name]).ravel())
            self._fh.write(f"{_fmt(time)},{name},{vals}\n")

    def log_summary(self, summary, bodies) -> None:
        """Log a ``StepSummary`` (its wrench rows are in body order)."""
        self.log_step(summary.time, {b.name: summary.wrench[i] for i, b in enumerate(bodies)
                                     if b.name in self.body_names})

    def close(self):
        self._fh.close()


class AsyncFrameWriter:
    """Frames of a running simulation without stalling it.

    ``submit(path, time, x, v=None)`` enqueues an asynchronous D2H copy of the
    device tensors into a pinned buffer (side stream, after the producing
    stream's work) and hands the file write to a background thread.  At most
    ``depth`` frames are in flight; ``close()`` drains them."""

    def __init__(self, depth: int = 2):
        self._q: queue.Queue = queue.Queue(maxsize=depth)
        self._stream = torch.cuda.Stream() if torch.cuda.is_available() else None
        self._err: list[BaseException] = []
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()

    def submit(self, path, time: float, x: torch.Tensor, v: torch.Tensor | None = None,
               producer: torch.cuda.Stream | None = None) -> None:
        if self._err:
            raise self._err[0]
        bufs = []
        ev = None
        if x.is_cuda:
            ready = torch.cuda.Event()
            ready.record(producer or torch.cuda.current_stream(x.device))
            with torch.cuda.stream(self._stream):
                self._stream.wait_event(ready)
                for t in (x, v):
                    if t is None:
                        bufs.append(None)
                        continue
                    h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
                    h.copy_(t, non_blocking=True)
                    bufs.append(h)
                ev = torch.cuda.Event()
                ev.record(self._stream)
        else:
            bufs = [x, v]
        self._q.put((Path(path), float(time), bufs, ev))

    def _run(self):
        while True:
            item = self._q.get()
            if item is None:
                return
            path, time, bufs, ev = item
            try:
                if ev is not None:
                    ev.synchronize()
                x, v = (None if b is None else b.numpy() for b in bufs)
                path.write_bytes(frame_bytes(time, x, v))
            except BaseException as e:  # surfaced on the next submit / close
                self._err.append(e)

    def close(self):
        self._q.put(None)
        self._t.join()
        if self._err:
            raise self._err[0]
