"""On-disk formats for real runs.

ragsim stores a workload as ``corpus.csv`` (doc_id, token_size, weight) and
``trace.jsonl`` (one request per line) (workload.py:203-259).  A real run also
needs the document embeddings the retrieval kernel scans, so a bundle adds
``embeddings.rcbemb`` next to them.  The format:

    offset 0   8 B  magic  b"RCBEMB01"
           8   4 B  dtype  1 = bf16 (the only dtype the tcgen05 scan reads)
          12   4 B  dim    (multiple of 64, <= 1024: the scan's 64-wide atoms)
          16   8 B  rows   (== corpus.csv's num_docs; row i is doc_id i)
          24   8 B  reserved (0)
          32   ...  rows x dim little-endian bf16, row-major (dim*2 bytes per row)

The header is 32 bytes, so the payload can be memory-mapped with numpy. A run
report can be extended with the B200 side of the run (swap GB/s, kernel times,
host core counts) next to ragsim's own report JSON (simulator.py:197-204).
"""

from __future__ import annotations

import json
import os
import platform
import struct

import numpy as np

MAGIC = b"RCBEMB01"
DTYPE_BF16 = 1
HEADER = struct.Struct("<8sIIQQ")  # magic, dtype, dim, rows, reserved
assert HEADER.size == 32


class FormatError(ValueError):
    """A bundle file does not match the format above."""


def _bf16_bits(emb) -> np.ndarray:
    """bf16 bit patterns (uint16 [rows, dim]) from a bf16 torch tensor or a float array
    (rounded to nearest even, as torch's .to(torch.bfloat16))."""
    try:
        import torch

        if isinstance(emb, torch.Tensor):
            t = emb.detach()
            if t.dtype != torch.bfloat16:
                t = t.to(torch.bfloat16)
            return t.cpu().contiguous().view(torch.int16).numpy().view(np.uint16)
    except ImportError:  # pragma: no cover - torch is part of the image
        pass
    a = np.ascontiguousarray(emb)
    if a.dtype == np.uint16:
        return a
    x = a.astype(np.float32).view(np.uint32)
    rounded = x + 0x7FFF + ((x >> 16) & 1)  # round to nearest even
    return (rounded >> 16).astype(np.uint16)


def write_embeddings(path: str, emb) -> None:
    bits = _bf16_bits(emb)
    if bits.ndim != 2:
        raise FormatError(f"embeddings must be 2-D, got shape {bits.shape}")
    rows, dim = bits.shape
    if dim % 64 != 0 or dim > 1024:
        raise FormatError(f"dim {dim} must be a multiple of 64 and <= 1024")
    with open(path, "wb") as fp:
        fp.write(HEADER.pack(MAGIC, DTYPE_BF16, dim, rows, 0))
        fp.write(bits.astype("<u2", copy=False).tobytes())


def read_header(path: str) -> tuple[int, int]:
    with open(path, "rb") as fp:
        raw = fp.read(HEADER.size)
    if len(raw) != HEADER.size:
        raise FormatError(f"{path}: truncated header")
    magic, dtype, dim, rows, _ = HEADER.unpack(raw)
    if magic != MAGIC:
        raise FormatError(f"{path}: bad magic {magic!r}")
    if dtype != DTYPE_BF16:
        raise FormatError(f"{path}: unsupported dtype code {dtype}")
    if dim == 0 or dim % 64 != 0 or dim > 1024:
        raise FormatError(f"{path}: bad dim {dim}")
    expect = HEADER.size + rows * dim * 2
    if os.path.getsize(path) != expect:
        raise FormatError(f"{path}: {os.path.getsize(path)} bytes, header says {expect}")
    return int(rows), int(dim)


def read_embeddings(path: str, rows: slice | None = None) -> np.ndarray:
    """uint16 bf16 bit patterns [rows, dim], memory-mapped (a row slice reads only it)."""
    n, dim = read_header(path)
    mm = np.memmap(path, dtype="<u2", mode="r", offset=HEADER.size, shape=(n, dim))
    return mm if rows is None else mm[rows]


def load_embeddings_device(path: str, device="cuda", chunk_rows: int = 1 << 18,
                           rows: slice | None = None):
    """bf16 [rows, dim] on the GPU (this rank's corpus shard with ``rows``), copied in
    pinned chunks so a 10M-row corpus never needs a second host copy."""
    import torch

    src = read_embeddings(path, rows)
    n, dim = src.shape
    out = torch.empty((n, dim), dtype=torch.bfloat16, device=device)
    stage = torch.empty((min(chunk_rows, max(n, 1)), dim), dtype=torch.int16).pin_memory()
    for r0 in range(0, n, chunk_rows):
        r1 = min(n, r0 + chunk_rows)
        stage[: r1 - r0].numpy()[:] = np.asarray(src[r0:r1]).view(np.int16)
        out[r0:r1].view(torch.int16).copy_(stage[: r1 - r0], non_blocking=True)
        torch.cuda.current_stream().synchronize()  # the stage buffer is reused
    return out


# ---------------------------------------------------------------------- bundles
def write_bundle(directory: str, corpus, trace, embeddings) -> dict:
    """corpus.csv + trace.jsonl (ragsim's own writers) + embeddings.rcbemb."""
    from ._ragsim import import_ragsim

    import_ragsim()
    from ragsim.workload import write_corpus, write_trace

    bits = _bf16_bits(embeddings)
    if bits.shape[0] != corpus.num_docs:
        raise FormatError(f"{bits.shape[0]} embedding rows for {corpus.num_docs} documents")
    os.makedirs(directory, exist_ok=True)
    paths = {"corpus": os.path.join(directory, "corpus.csv"),
             "trace": os.path.join(directory, "trace.jsonl"),
             "embeddings": os.path.join(directory, "embeddings.rcbemb")}
    write_corpus(corpus, paths["corpus"])
    write_trace(trace, paths["trace"])
    write_embeddings(paths["embeddings"], bits)
    return paths


def read_bundle(directory: str):
    """(corpus, trace, embeddings uint16 memmap) with the cross-file checks a run needs:
    one embedding row per document, every requested document in the corpus."""
    from ._ragsim import import_ragsim

    import_ragsim()
    from ragsim.workload import read_corpus, read_trace

    corpus = read_corpus(os.path.join(directory, "corpus.csv"))
    trace = read_trace(os.path.join(directory, "trace.jsonl"))
    emb = read_embeddings(os.path.join(directory, "embeddings.rcbemb"))
    if emb.shape[0] != corpus.num_docs:
        raise FormatError(f"{emb.shape[0]} embedding rows for {corpus.num_docs} documents")
    bad = [r.id for r in trace for d in r.doc_sequence if not 0 <= d < corpus.num_docs]
    if bad:
        raise FormatError(f"requests {bad[:5]} reference documents outside the corpus")
    return corpus, trace, emb


# ---------------------------------------------------------------------- reports
def host_info() -> dict:
    cpu = platform.processor() or ""
    try:
        with open("/proc/cpuinfo") as fp:
            for line in fp:
                if line.startswith("model name"):
                    cpu = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cpu_model": cpu, "cores_usable": len(os.sched_getaffinity(0)),
            "cores_total": os.cpu_count()}


def extend_report(report_json: str, *, kernels: dict | None = None, swap: dict | None = None,
                  gpu: str | None = None) -> str:
    """ragsim's report JSON (SimReport.to_json, simulator.py:197-204) plus a "b200" block:
    measured swap GB/s, kernel times and the host the decisions ran on.  The reference's
    own keys are untouched, so its readers keep working."""
    payload = json.loads(report_json)
    if "b200" in payload:
        raise FormatError("report already extended")
    payload["b200"] = {"host": host_info(), "gpu": gpu, "swap": swap or {},
                       "kernels": kernels or {}}
    return json.dumps(payload, sort_keys=True, indent=2)
