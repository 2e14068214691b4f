"""GPU ingestion: the CSR build of
``Dataset.from_token_lists`` (reference core.py:60-95) and the SPEC
harness's text loader / pair writer, on the
sm_100a kernels of csrc/ingest.cu.

  from_token_lists(lists, d=None, source_lines=None) -> Dataset
  from_flat(values, offsets, d=None, source_lines=None) -> Dataset
  load_dataset(path, d=None) -> Dataset       (source_lines = 1-based lines)
  write_pairs(path, a, b, similarity)          ("idA idB sim", 6 decimals)

Results equal the reference's from_token_lists on the same input (golden
fixtures made by the reference, tests/golden/ingest_*.npz).  Errors follow
the reference: tokens outside [0, d) with d given raise ValueError
("column index exceeds matrix dimensions"); a non-integer field raises
ValueError naming its line.
"""
from __future__ import annotations

import ctypes
import itertools

import numpy as np

from .core import Dataset


def _finish(ctx, st, stream, source_lines):
    n, nnz = int(st.n_sets), int(st.nnz)
    tokens = np.empty(nnz, dtype=np.uint32)
    offsets = np.zeros(n + 1, dtype=np.int64)
    src = np.empty(n, dtype=np.int64)
    ctx.check(ctx.lib.cpsj_ingest_copy(ctx.handle, tokens.ctypes.data, offsets.ctypes.data, src.ctypes.data,
                                       stream))
    lines = None
    if source_lines is not None:
        sl = np.asarray(source_lines)
        lines = [int(x) for x in sl[src]] if n else []
    if n == 0:
        return Dataset([], int(st.d), source_lines=[] if source_lines is not None else None)
    return Dataset(d=int(st.d), source_lines=lines, _csr=(tokens, offsets))


def from_flat(values, offsets, d: int | None = None, source_lines=None) -> Dataset:
    """from_token_lists over records given as one int64 array + offsets."""
    import torch

    from ._native import Context, IngestStats
    ctx = Context.get()
    dev = torch.device("cuda", ctx.device)
    stream = torch.cuda.current_stream(dev).cuda_stream
    vals = np.ascontiguousarray(values, dtype=np.int64)
    offs = np.ascontiguousarray(offsets, dtype=np.int64)
    n = len(offs) - 1
    d_vals = torch.from_numpy(vals).to(dev) if len(vals) else torch.zeros(1, dtype=torch.int64, device=dev)
    d_offs = torch.from_numpy(offs).to(dev)
    st = IngestStats()
    ctx.check(ctx.lib.cpsj_ingest_lists(ctx.handle, d_vals.data_ptr(), d_offs.data_ptr(), n,
                                        -1 if d is None else int(d), ctypes.byref(st), stream))
    return _finish(ctx, st, stream, source_lines)


def from_token_lists(token_lists, d: int | None = None, source_lines=None) -> Dataset:
    """Dataset.from_token_lists (core.py:60-95) with the sort / unique /
    drop / dedup / remap work on the GPU; the host only flattens the lists."""
    lens = [len(r) for r in token_lists] if not isinstance(token_lists, np.ndarray) else None
    if lens is None:
        token_lists = list(token_lists)
        lens = [len(r) for r in token_lists]
    offs = np.zeros(len(lens) + 1, dtype=np.int64)
    np.cumsum(lens, out=offs[1:])
    vals = np.fromiter(itertools.chain.from_iterable(token_lists), dtype=np.int64, count=int(offs[-1]))
    return from_flat(vals, offs, d, source_lines)


def load_dataset(path: str, d: int | None = None) -> Dataset:
    """SPEC load_dataset: one record per line of blank-separated decimal
    tokens; parsed, cleaned and densely remapped on the GPU.  source_lines
    holds the 1-based line number of every kept record; an empty file gives
    an empty dataset."""
    import torch

    from ._native import Context, IngestStats
    ctx = Context.get()
    dev = torch.device("cuda", ctx.device)
    stream = torch.cuda.current_stream(dev).cuda_stream
    raw = np.fromfile(path, dtype=np.uint8)
    d_raw = torch.from_numpy(raw).to(dev) if len(raw) else torch.zeros(1, dtype=torch.uint8, device=dev)
    st = IngestStats()
    ctx.check(ctx.lib.cpsj_parse_text(ctx.handle, d_raw.data_ptr(), len(raw), -1 if d is None else int(d),
                                      ctypes.byref(st), stream))
    lines = np.arange(1, int(st.n_input_records) + 1, dtype=np.int64)
    return _finish(ctx, st, stream, lines)


def write_pairs(path: str, a, b, similarity) -> None:
    """Output pairs one per line, "idA idB similarity" with 6 decimals
    (SPEC:575)."""
    a = np.asarray(a, dtype=np.int64)
    b = np.asarray(b, dtype=np.int64)
    s = np.asarray(similarity, dtype=np.float64)
    with open(path, "w") as f:
        f.writelines(f"{x} {y} {v:.6f}\n" for x, y, v in zip(a.tolist(), b.tolist(), s.tolist()))
