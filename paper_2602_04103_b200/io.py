"""Host-side input preparation for real data: ASCII DNA -> symbol codes -> 2-bit packed words,
FASTA / FASTQ readers.  Vectorised numpy (no per-character Python loop); not on the hot path.

Codes follow DESIGN.md reading R1: A=0, C=1, G=2, T=3 (case-insensitive).  Any other
character (N, IUPAC codes, ...) is rejected unless ``replace_invalid`` gives a code to use
(SPEC S:375 rejects such reads; many aligners map N to a fixed base instead).
"""
from __future__ import annotations

import numpy as np

_LUT = np.full(256, 255, dtype=np.uint8)
for _ch, _v in zip(b"ACGTacgt", (0, 1, 2, 3, 0, 1, 2, 3)):
    _LUT[_ch] = _v


def encode(seq: bytes | str | np.ndarray, replace_invalid: int | None = None) -> np.ndarray:
    """ASCII DNA -> uint8 codes 0..3."""
    if isinstance(seq, str):
        seq = seq.encode()
    raw = np.frombuffer(seq, dtype=np.uint8) if not isinstance(seq, np.ndarray) else seq.astype(np.uint8)
    codes = _LUT[raw]
    bad = codes == 255
    if bad.any():
        if replace_invalid is None:
            i = int(np.argmax(bad))
            raise ValueError(f"non-ACGT character {chr(raw[i])!r} at position {i}")
        codes = np.where(bad, np.uint8(replace_invalid), codes)
    return codes


def decode(codes: np.ndarray) -> str:
    return np.frombuffer(b"ACGT", dtype=np.uint8)[np.asarray(codes, dtype=np.uint8)].tobytes().decode()


def pack2(codes: np.ndarray) -> np.ndarray:
    """uint8 codes -> 2-bit little-endian packed uint64 words (char i at bits 2(i%32) of word i/32)."""
    codes = np.asarray(codes, dtype=np.uint8)
    n = codes.size
    pad = np.zeros(((n + 31) // 32) * 32, dtype=np.uint64)
    pad[:n] = codes
    pad = pad.reshape(-1, 32) << (2 * np.arange(32, dtype=np.uint64))
    out = np.bitwise_or.reduce(pad, axis=1) if pad.size else np.zeros(0, np.uint64)
    return np.ascontiguousarray(np.concatenate([out, np.zeros(1, np.uint64)]))   # one spare word


def unpack2(words: np.ndarray, n: int) -> np.ndarray:
    b = np.asarray(words, dtype=np.uint64).view(np.uint8)
    sym = np.stack([(b >> (2 * k)) & 3 for k in range(4)], axis=1).reshape(-1)
    return sym[:n].astype(np.uint8)


def reverse_complement(codes: np.ndarray) -> np.ndarray:
    """A<->T, C<->G, reversed."""
    return (3 - np.asarray(codes, dtype=np.uint8)[::-1]).astype(np.uint8)


def read_fasta(path: str, replace_invalid: int | None = None) -> list[tuple[str, np.ndarray]]:
    """All records of a FASTA file as (name, codes)."""
    recs, name, chunks = [], None, []
    with open(path, "rb") as f:
        for line in f:
            line = line.rstrip(b"\r\n")
            if line.startswith(b">"):
                if name is not None:
                    recs.append((name, encode(b"".join(chunks), replace_invalid)))
                name, chunks = line[1:].decode().split()[0] if len(line) > 1 else "", []
            elif line:
                chunks.append(line)
    if name is not None:
        recs.append((name, encode(b"".join(chunks), replace_invalid)))
    return recs


def read_fastq(path: str, replace_invalid: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """Reads of a FASTQ file as (concatenated codes, u32 lengths) — the qr_fm_count input form."""
    seqs = []
    with open(path, "rb") as f:
        while True:
            h = f.readline()
            if not h:
                break
            s = f.readline().rstrip(b"\r\n")
            f.readline()
            f.readline()
            seqs.append(s)
    lens = np.array([len(s) for s in seqs], dtype=np.uint32)
    cat = encode(b"".join(seqs), replace_invalid) if seqs else np.zeros(0, np.uint8)
    return np.ascontiguousarray(np.concatenate([cat, np.zeros(8, np.uint8)])), lens
