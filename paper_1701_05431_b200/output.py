"""Asynchronous solution output (the paper's gatherForOutput -> switch ->
outputToDisk pipeline) on top of fv2d_snapshot.

The device side (conversion into a staging buffer on a side stream, D2H into
page-locked memory) overlaps the following time steps; this module adds the
host side: a background writer thread that waits for each snapshot and writes
it in SPEC's solution format: magic "TFV1", Nx, Ny, nVar as
little-endian int64, t as float64, then Nx*Ny*nVar float64 with x fastest and
the variable innermost (the paper's Cell order).
"""
from __future__ import annotations

import queue
import struct
import threading

import numpy as np

from . import fv2d

MAGIC = b"TFV1"


def write_tfv1(path: str, W: np.ndarray, t: float) -> None:
    ny, nx, nv = W.shape
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<qqqd", nx, ny, nv, float(t)))
        f.write(np.ascontiguousarray(W, dtype="<f8").tobytes())


def read_tfv1(path: str):
    with open(path, "rb") as f:
        if f.read(4) != MAGIC:
            raise ValueError(f"{path}: not a TFV1 file")
        nx, ny, nv, t = struct.unpack("<qqqd", f.read(32))
        W = np.frombuffer(f.read(), dtype="<f8").reshape(ny, nx, nv).copy()
    return W, t


class AsyncWriter:
    """Snapshots of a Solver written to disk by a background thread.

    >>> w = AsyncWriter(solver, "out_{step:06d}.tfv1", nbuf=2)
    >>> for k in range(60):
    ...     solver.step(dt); t += dt
    ...     if (k + 1) % 20 == 0: w.submit(k + 1, t)
    >>> w.close()

    `nbuf` page-locked buffers rotate; submit() blocks only when all are still
    being written.  Stepping is never blocked by disk I/O."""

    def __init__(self, solver: "fv2d.Solver", pattern: str | None, nbuf: int = 2):
        """pattern None: snapshots are taken but not written (to time the device
        and PCIe side of the pipeline without the disk)."""
        self.solver = solver
        self.pattern = pattern
        self.free = queue.Queue()
        for _ in range(max(1, nbuf)):
            self.free.put(fv2d.PinnedArray(solver._shape(fv2d.AOS)))
        self.todo = queue.Queue()
        self.written = []
        self.error = None
        self.thread = threading.Thread(target=self._run, daemon=True)
        self.thread.start()

    def submit(self, step: int, t: float) -> None:
        buf = self.free.get()
        self.solver.snapshot(buf, fv2d.AOS)
        self.todo.put((buf, step, t))

    def _run(self):
        while True:
            item = self.todo.get()
            if item is None:
                return
            buf, step, t = item
            try:
                self.solver.snapshot_wait()
                if self.pattern is not None:
                    path = self.pattern.format(step=step)
                    write_tfv1(path, buf.array, t)
                    self.written.append(path)
                else:
                    self.written.append(None)
            except Exception as e:  # reported by close()
                self.error = e
            finally:
                self.free.put(buf)

    def close(self):
        self.todo.put(None)
        self.thread.join()
        while not self.free.empty():
            self.free.get().free()
        if self.error:
            raise self.error
        return self.written
