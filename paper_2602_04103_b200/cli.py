"""Command line front end (the SPEC's `quadfm count`, on real files).

  python -m paper_2602_04103_b200.cli fm-count --fasta genome.fa --fastq reads.fq \
         [--both-strands] [--max-mismatches 0-3] [--out counts.tsv]

Builds the QuadFm index of the FASTA records (concatenated in file order; matches spanning
two records are counted like any other substring) on the GPU and writes one line per read:
name-less index, forward count[, reverse-complement count].
"""
from __future__ import annotations

import argparse
import sys
import time

import numpy as np


def _fm_count(args) -> int:
    import torch

    from . import (QR_LAYOUT_QUADRANK16, QR_LAYOUT_QUADRANK16X2, io, qr_fm_build, qr_fm_count_approx,
                   qr_fm_count_approx_both, qr_fm_count_both, qr_sync)

    t0 = time.perf_counter()
    recs = io.read_fasta(args.fasta, replace_invalid=args.replace_invalid)
    text = np.concatenate([r[1] for r in recs]) if recs else np.zeros(0, np.uint8)
    n = int(text.size)
    if n == 0:
        print("empty FASTA", file=sys.stderr)
        return 2
    cat, lens = io.read_fastq(args.fastq, replace_invalid=args.replace_invalid)
    m = int(lens.size)
    t1 = time.perf_counter()
    layout = QR_LAYOUT_QUADRANK16X2 if args.bwt_layout == "quadrank16x2" else QR_LAYOUT_QUADRANK16
    fm = qr_fm_build(io.pack2(text), n, device=args.device, bwt_layout=layout)
    t2 = time.perf_counter()
    dev = torch.device("cuda", args.device)
    dcat, dlens = torch.from_numpy(cat).to(dev), torch.from_numpy(lens).to(dev)
    fwd = torch.empty(m, dtype=torch.int32, device=dev)
    rc = torch.empty(m, dtype=torch.int32, device=dev) if args.both_strands else None
    if args.max_mismatches and rc is not None:
        qr_fm_count_approx_both(fm, dcat, dlens, 0, args.max_mismatches, fwd, rc, m)
    elif args.max_mismatches:
        qr_fm_count_approx(fm, dcat, dlens, 0, args.max_mismatches, fwd, m)
    elif rc is not None:
        qr_fm_count_both(fm, dcat, dlens, 0, fwd, rc, m)
    else:
        from . import qr_fm_count

        qr_fm_count(fm, dcat, dlens, 0, fwd, m)
    qr_sync()
    t3 = time.perf_counter()
    f = fwd.cpu().numpy().view(np.uint32)
    r = rc.cpu().numpy().view(np.uint32) if rc is not None else None
    out = open(args.out, "w") if args.out else sys.stdout
    for i in range(m):
        out.write(f"{i}\t{f[i]}" + (f"\t{r[i]}\n" if r is not None else "\n"))
    if args.out:
        out.close()
    print(f"text {n} bp, {m} reads: read {t1 - t0:.2f}s, build {t2 - t1:.2f}s, count {t3 - t2:.3f}s",
          file=sys.stderr)
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="qrank")
    sub = ap.add_subparsers(dest="cmd", required=True)
    f = sub.add_parser("fm-count", help="count reads in a genome (QuadFm)")
    f.add_argument("--fasta", required=True)
    f.add_argument("--fastq", required=True)
    f.add_argument("--both-strands", action="store_true")
    f.add_argument("--max-mismatches", type=int, default=0, choices=[0, 1, 2, 3])
    f.add_argument("--replace-invalid", type=int, default=None, help="code for non-ACGT characters (default: reject)")
    f.add_argument("--device", type=int, default=0)
    f.add_argument("--bwt-layout", default="quadrank16", choices=["quadrank16", "quadrank16x2"],
                   help="rank layout of the BWT: the paper's QuadRank16 (2.29 bits/bp) or the sector-local "
                        "QuadRank16x2 (2.67 bits/bp, faster on L2-resident indexes)")
    f.add_argument("--out", default=None)
    args = ap.parse_args(argv)
    if args.cmd == "fm-count":
        return _fm_count(args)
    return 1


if __name__ == "__main__":
    sys.exit(main())
