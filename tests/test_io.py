"""Host-side input preparation (paper_2602_04103_b200.io): encoding, 2-bit packing (the layout
the generators and the C ABI use), FASTA / FASTQ reading, reverse complement."""
import numpy as np
import pytest

import gen
from paper_2602_04103_b200 import io


def test_encode_pack_roundtrip():
    s = "ACGTacgtTTGA"
    c = io.encode(s)
    assert list(c) == [0, 1, 2, 3, 0, 1, 2, 3, 3, 3, 2, 0]
    assert io.decode(c) == s.upper()
    w = io.pack2(io.encode("ACGT"))
    assert int(w[0]) & 0xFF == 0b11100100                      # pack_quad([0,1,2,3])
    n = 100003
    words = gen.dna(5, n)
    sym = gen.unpack_dna(words, n)
    assert np.array_equal(io.pack2(sym)[: words.size], words)   # same layout as the generators / ABI
    assert np.array_equal(io.unpack2(io.pack2(sym), n), sym)
    with pytest.raises(ValueError):
        io.encode("ACGN")
    assert list(io.encode("ACGN", replace_invalid=0)) == [0, 1, 2, 0]
    assert list(io.reverse_complement(np.array([0, 1], np.uint8))) == [2, 3]
    r = np.random.default_rng(1).integers(0, 4, 1000).astype(np.uint8)
    assert np.array_equal(io.reverse_complement(io.reverse_complement(r)), r)


def test_fasta_fastq(tmp_path):
    fa = tmp_path / "g.fa"
    fa.write_text(">chr1 desc\nACGT\nTTGG\n>chr2\nGGCC\n")
    recs = io.read_fasta(str(fa))
    assert [r[0] for r in recs] == ["chr1", "chr2"]
    assert io.decode(recs[0][1]) == "ACGTTTGG" and io.decode(recs[1][1]) == "GGCC"
    fq = tmp_path / "r.fq"
    fq.write_text("@r1\nACG\n+\nIII\n@r2\nTTTT\n+\nIIII\n")
    cat, lens = io.read_fastq(str(fq))
    assert list(lens) == [3, 4]
    assert io.decode(cat[:7]) == "ACGTTTT"
