"""Streaming GPU -> file writers for the reference's on-disk formats
(SURVEY.md 8(f) row 4), so disputes can be served from a committed trace:

  * NAOT tensor files      tensor.py:146-180   (magic, u32 version, u8 dtype code,
                                                u32 rank, rank x u64 dims, LE payload)
  * trace dumps            engine.py:449-478   (<i:06d>.naot per node + manifest.json)
  * bound dumps            bounds.py:265-282   (FP64 NAOT per node + manifest.json)

`NaotWriter` moves device tensors through a ring of pinned staging slots:
the D2H copy of slot k runs on a copy stream while a worker thread writes slot
k-1 to disk, so the GPU never waits for the file system and the caller never
synchronizes (the writer keeps each source tensor alive on the copy stream
until its bytes have left the device).  `TraceWriter` / `BoundWriter` plug
into `executor.StreamingVerifier.run(..., trace_writer=...)`; `TraceReader`
loads node tensors back onto the device for re-execution.
Files are byte-identical to the reference's writers (tests/golden/ref_traceio.json).
"""

from __future__ import annotations

import json
import queue
import struct
import threading
from pathlib import Path

import numpy as np
import torch

from .tensor import TENSOR_FILE_VERSION, TENSOR_MAGIC, read_tensor_file

_CODES = {torch.float32: 0, torch.float64: 1}


def naot_header(shape, dtype: torch.dtype) -> bytes:
    """tensor.py:146-161 header bytes."""
    if dtype not in _CODES:
        raise ValueError(f"unsupported dtype {dtype}")
    h = TENSOR_MAGIC + struct.pack("<IBI", TENSOR_FILE_VERSION, _CODES[dtype], len(shape))
    for d in shape:
        h += struct.pack("<Q", int(d))
    return h


class NaotWriter:
    """Asynchronous NAOT writer: pinned staging ring + copy stream + one
    writer thread.  submit() returns immediately; close() waits for the disk."""

    def __init__(self, device=None, slots: int = 3, slot_bytes: int = 64 << 20):
        self.dev = torch.device(device) if device is not None else torch.device("cuda")
        self.stream = torch.cuda.Stream(self.dev)
        self.slot_bytes = int(slot_bytes)
        self._slots = [torch.empty(self.slot_bytes, dtype=torch.uint8).pin_memory()
                       for _ in range(max(2, slots))]
        self._free = [threading.Event() for _ in self._slots]
        for e in self._free:
            e.set()
        self._next = 0
        self._q: queue.Queue = queue.Queue()
        self._err: BaseException | None = None
        self._thread = threading.Thread(target=self._run, daemon=True)
        self._thread.start()
        self.bytes_written = 0

    # ----------------------------------------------------------- worker
    def _run(self):
        fh = None
        while True:
            item = self._q.get()
            if item is None:
                break
            op = item[0]
            try:
                if op == "open":
                    fh = open(item[1], "wb")
                    fh.write(item[2])
                elif op == "chunk":
                    _, k, n, ev = item
                    ev.synchronize()
                    fh.write(memoryview(self._slots[k].numpy())[:n])
                    self.bytes_written += n
                    self._free[k].set()
                elif op == "close":
                    fh.close()
                    fh = None
                elif op == "sync":
                    item[1].set()
            except BaseException as exc:  # surfaced by flush()/close()
                self._err = exc
                if op == "chunk":
                    self._free[item[1]].set()

    # ------------------------------------------------------------- API
    def submit(self, path, t: torch.Tensor) -> None:
        """Queue tensor t (FP32/FP64; CUDA or host) for writing as a NAOT file."""
        if self._err:
            raise self._err
        if t.dtype not in _CODES:
            raise ValueError(f"unsupported dtype {t.dtype}")
        shape = tuple(t.shape)
        self._q.put(("open", str(path), naot_header(shape, t.dtype)))
        flat = t.contiguous().reshape(-1).view(torch.uint8)
        nbytes = flat.numel()
        if nbytes == 0:
            self._q.put(("close",))
            return
        if flat.is_cuda:
            self.stream.wait_stream(torch.cuda.current_stream(flat.device))
        off = 0
        while off < nbytes:
            k = self._next
            self._next = (self._next + 1) % len(self._slots)
            self._free[k].wait()
            self._free[k].clear()
            n = min(self.slot_bytes, nbytes - off)
            with torch.cuda.stream(self.stream):
                self._slots[k][:n].copy_(flat[off:off + n], non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(self.stream)
            self._q.put(("chunk", k, n, ev))
            off += n
        if flat.is_cuda:
            flat.record_stream(self.stream)
        self._q.put(("close",))

    def flush(self) -> None:
        done = threading.Event()
        self._q.put(("sync", done))
        done.wait()
        if self._err:
            raise self._err

    def close(self) -> None:
        self.flush()
        self._q.put(None)
        self._thread.join()


class TraceWriter:
    """engine.py:449-464 save_trace, streamed: write(i, tensor) per node as it
    is produced, close() writes the manifest."""

    def __init__(self, dirpath, profile_id: str, input_digests: dict, weight_digests: dict,
                 device=None, writer: NaotWriter | None = None):
        self.dir = Path(dirpath)
        self.dir.mkdir(parents=True, exist_ok=True)
        self.profile_id = profile_id
        self.input_digests = dict(input_digests)
        self.weight_digests = dict(weight_digests)
        self.writer = writer or NaotWriter(device)
        self.n_nodes = 0

    def write(self, i: int, t: torch.Tensor) -> None:
        self.writer.submit(self.dir / f"{i:06d}.naot", t)
        self.n_nodes = max(self.n_nodes, i + 1)

    def close(self, n_nodes: int | None = None) -> None:
        self.writer.close()
        manifest = {"n_nodes": int(n_nodes if n_nodes is not None else self.n_nodes),
                    "profile_id": self.profile_id,
                    "input_digests": self.input_digests,
                    "weight_digests": self.weight_digests}
        with open(self.dir / "manifest.json", "w") as fh:
            json.dump(manifest, fh, sort_keys=True, indent=1)


class BoundWriter:
    """bounds.py:265-282 save_bounds, streamed: FP64 tensor files + manifest
    (FP32 rounded-up streaming bounds are widened to FP64 on the device)."""

    def __init__(self, dirpath, model, profile_id: str, device=None,
                 writer: NaotWriter | None = None):
        self.dir = Path(dirpath)
        self.dir.mkdir(parents=True, exist_ok=True)
        self.model, self.profile_id = model, profile_id
        self.writer = writer or NaotWriter(device)
        self.n_nodes = 0

    def write(self, i: int, eps: torch.Tensor) -> None:
        e = eps if eps.dtype == torch.float64 else eps.double()
        self.writer.submit(self.dir / f"{i:06d}.naot", e)
        self.n_nodes = max(self.n_nodes, i + 1)

    def close(self, n_nodes: int | None = None) -> None:
        self.writer.close()
        manifest = {"n_nodes": int(n_nodes if n_nodes is not None else self.n_nodes),
                    "profile_id": self.profile_id,
                    "fp_model": {"u": self.model.u, "lambda": self.model.lam,
                                 "mode": self.model.mode}}
        with open(self.dir / "manifest.json", "w") as fh:
            json.dump(manifest, fh, sort_keys=True, indent=1)


class TraceReader:
    """engine.py:467-478 load_trace, lazily: node(i) -> device tensor."""

    def __init__(self, dirpath):
        self.dir = Path(dirpath)
        with open(self.dir / "manifest.json") as fh:
            self.manifest = json.load(fh)
        self.n_nodes = int(self.manifest["n_nodes"])
        self.profile_id = self.manifest.get("profile_id")

    def node(self, i: int, device="cuda") -> torch.Tensor:
        arr = read_tensor_file(self.dir / f"{i:06d}.naot")
        host = torch.from_numpy(np.ascontiguousarray(arr))
        if torch.device(device).type == "cuda":
            host = host.pin_memory()
            return host.to(device, non_blocking=True)
        return host


def save_trace(dirpath, trace, device=None) -> None:
    """engine.py:449-464 (drop-in; device tensors stream through the writer)."""
    w = TraceWriter(dirpath, trace.profile_id, trace.input_digests, trace.weight_digests, device)
    for i, t in enumerate(trace.tensors):
        w.write(i, _as_tensor(t))
    w.close(len(trace.tensors))


def load_trace(dirpath):
    """engine.py:467-478 (drop-in)."""
    from .engine_trace import Trace
    from .tensor import Tensor
    r = TraceReader(dirpath)
    tensors = []
    for i in range(r.n_nodes):
        arr = read_tensor_file(r.dir / f"{i:06d}.naot")
        tensors.append(Tensor(arr.shape, arr.reshape(-1)))
    return Trace(tensors=tensors, profile_id=r.manifest["profile_id"],
                 input_digests=r.manifest["input_digests"],
                 weight_digests=r.manifest["weight_digests"])


def _as_tensor(t) -> torch.Tensor:
    if isinstance(t, torch.Tensor):
        return t
    dev = getattr(t, "_dev", None)
    if dev is not None:
        return dev.reshape(tuple(t.shape))
    return torch.from_numpy(np.ascontiguousarray(np.asarray(t.array, np.float32)))
