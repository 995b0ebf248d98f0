"""Host feature ingestion: PTX text and DCGM CSV traces into the
arrays the device feature stage consumes.

parse_ptx / load_dcgm_samples mirror the reference functions of the same names
(ptx_features.cpp:238-309, telemetry.cpp:63-101); the work is done by the
library's host C++ (csrc/ingest.cpp), which releases the GIL, so many files parse
in parallel on a thread pool (ingest_corpus)."""

from __future__ import annotations

import ctypes as C
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from ._lib import DsoError, ErrorKind, lib

ROWS = 126  # instr 101 | dtype 17 | memspace 8


def _parse(text: str | bytes):
    data = text.encode() if isinstance(text, str) else bytes(text)
    h = C.c_void_p()
    msg = C.create_string_buffer(512)
    st = lib().dso_ptx_parse(data, len(data), C.byref(h), msg, 512)
    if st:
        raise DsoError(ErrorKind(st - 1), msg.value.decode())
    return h


def parse_ptx(text: str | bytes):
    """[(kernel_name, counts uint64[126], total_instructions)] in source order."""
    L = lib()
    h = _parse(text)
    try:
        out = []
        for k in range(L.dso_ptx_kernel_count(h)):
            c = np.zeros(ROWS, np.uint64)
            tot = C.c_uint64()
            L.dso_ptx_kernel_counts(h, k, c.ctypes.data, C.byref(tot))
            out.append((L.dso_ptx_kernel_name(h, k).decode(), c, int(tot.value)))
        return out
    finally:
        L.dso_ptx_free(h)


def ptx_csr(text: str | bytes):
    """(names, row_ptr uint64[n+1], entries uint32[nnz]) of one PTX file, the sparse
    count input of dso_pipeline_csr."""
    L = lib()
    h = _parse(text)
    try:
        n = L.dso_ptx_kernel_count(h)
        rp = np.zeros(n + 1, np.uint64)
        ent = np.zeros(max(L.dso_ptx_nnz(h), 1), np.uint32)
        st = L.dso_ptx_csr(h, rp.ctypes.data, ent.ctypes.data)
        if st:
            raise DsoError(ErrorKind(st - 1), "a category count does not fit the CSR entry")
        names = [L.dso_ptx_kernel_name(h, k).decode() for k in range(n)]
        return names, rp, ent[: int(rp[-1])]
    finally:
        L.dso_ptx_free(h)


def load_dcgm_samples(text: str | bytes) -> np.ndarray:
    """Per-metric means [smact, smocc, tenso, drama, fp64a, fp32a, fp16a, intac]."""
    data = text.encode() if isinstance(text, str) else bytes(text)
    out = np.zeros(8)
    msg = C.create_string_buffer(512)
    st = lib().dso_load_dcgm_csv(data, len(data), out.ctypes.data, msg, 512)
    if st:
        raise DsoError(ErrorKind(st - 1), msg.value.decode())
    return out


def ingest_corpus(ptx_texts, dcgm_texts, threads: int = 8):
    """One kernel per (PTX file's first kernel, DCGM trace) pair, parsed in parallel:
    (names, row_ptr uint64[n+1], entries uint32, dcgm float32[8, n]) ready for
    Context.pipeline_csr (host path)."""
    if len(ptx_texts) != len(dcgm_texts):
        raise DsoError(ErrorKind.InvalidArgument, "ptx and dcgm lists differ in length")
    with ThreadPoolExecutor(max(1, threads)) as ex:
        csr = list(ex.map(ptx_csr, ptx_texts))
        dc = list(ex.map(load_dcgm_samples, dcgm_texts))
    names, rows, ents = [], [0], []
    for nm, rp, ent in csr:
        if len(nm) == 0:
            raise DsoError(ErrorKind.MalformedPtx, "no .entry kernel in a PTX file")
        names.append(nm[0])
        e = ent[int(rp[0]):int(rp[1])]
        ents.append(e)
        rows.append(rows[-1] + len(e))
    row_ptr = np.array(rows, np.uint64)
    entries = np.concatenate(ents).astype(np.uint32) if ents else np.zeros(1, np.uint32)
    dcgm = np.ascontiguousarray(np.array(dc, np.float64).T.astype(np.float32))
    return names, row_ptr, entries, dcgm
