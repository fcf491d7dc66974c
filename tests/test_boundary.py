"""The C-ABI boundary without a GPU: the library loads, exports every
function include/spb_b200.h declares, and its integer-exact host code (suffix
rule, chunk layout, contributor sets, batch draws, worker placement,
synthetic data) is bit-exact with the CPU oracle."""
import os
import re

import numpy as np
import pytest

from conftest import ROOT
from paper_2111_10672_b200 import spb


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "spb_b200.h")).read()
    return sorted(set(re.findall(r"SPB_API\s+[\w\s\*]*?\b(spb_\w+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    lib = spb.load_library()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(spb.EXPORTED) == syms


def test_exports_match_nm():
    import subprocess

    out = subprocess.run(["nm", "-D", "--defined-only", spb.LIB_PATH], capture_output=True, text=True).stdout
    exported = sorted(l.split()[-1] for l in out.splitlines() if " T spb_" in l)
    assert exported == header_symbols()


def test_suffix_rule_kats():
    assert spb.suffix_layers(3, 3, 9) == 9
    assert spb.suffix_layers(1, 3, 9) == 3
    assert spb.suffix_layers(2, 3, 9) == 6
    assert spb.suffix_layers(1, 4, 10) == 3
    with pytest.raises(spb.ArgumentError):
        spb.suffix_layers(0, 3, 9)
    with pytest.raises(spb.ArgumentError):
        spb.suffix_layers(4, 3, 9)
    with pytest.raises(spb.ArgumentError):
        spb.chunk_coverage(0, 4)
    with pytest.raises(spb.ArgumentError):
        spb.chunk_coverage(5, 4)
    assert spb.chunk_layout(3, 7) == [(1, 2), (3, 4), (5, 7)]


def test_bookkeeping_exhaustive_vs_oracle(orc):
    # Every (k, L) up to 64 x 64: suffix rule, chunk layout, contributor counts.
    for k in range(1, 65):
        for L in range(1, 65):
            assert spb.layer_chunks(k, L) == orc.layer_chunks(k, L)
            assert spb.chunk_layout(k, L) == orc.chunk_layout(k, L)
            for j in (1, (k + 1) // 2, k):
                assert spb.suffix_layers(j, k, L) == orc.suffix_layers(j, k, L)
    for k in range(1, 17):
        for m in range(1, k + 1):
            assert spb.chunk_coverage(m, k) == orc.chunk_coverage(m, k)


def test_coverage_law():
    # verify.cpp:186-215: chunk m has m contributors; each worker's chunks add up to its suffix.
    for k in range(1, 17):
        for L in (k, 2 * k, 3 * k + 1, max(1, 2 * k - 1)):
            spans = spb.chunk_layout(k, L)
            per_layer = [0] * L
            for j in range(1, k + 1):
                s = spb.suffix_layers(j, k, L)
                for l in range(L - s + 1, L + 1):
                    per_layer[l - 1] += 1
            assert spb.layer_chunks(k, L) == per_layer
            for j in range(1, k + 1):
                covered = sum(last - first + 1 for m, (first, last) in enumerate(spans, 1)
                              if j >= k - m + 1 and last >= first)
                assert covered == spb.suffix_layers(j, k, L)


def test_draw_batch_vs_oracle(orc):
    for seed, step, worker, n in [(11, 1, 1, 4096), (11, 7, 8, 8192), (2**40 + 3, 123, 4, 60000), (0, 0, 0, 1)]:
        assert (spb.draw_batch(seed, step, worker, 257, n) == orc.draw_batch(seed, step, worker, 257, n)).all()


@pytest.mark.parametrize("k,L,nr", [(8, 16, 1), (8, 16, 2), (8, 16, 4), (8, 16, 8), (4, 3, 2), (6, 12, 4), (5, 7, 3)])
def test_rank_workers_partition(k, L, nr):
    owned = [spb.rank_workers(k, L, r, nr) for r in range(nr)]
    assert sorted(sum(owned, [])) == list(range(1, k + 1))
    sizes = [len(o) for o in owned]
    assert max(sizes) - min(sizes) <= 1
    for o in owned:
        assert o == sorted(o)
    if nr == k:
        assert owned == [[j] for j in range(1, k + 1)]  # one worker per rank
    elif nr >= 4:  # default from 4 ranks: contiguous blocks of workers (fewer exchange bytes)
        assert sum(owned, []) == list(range(1, k + 1))
    elif k % (2 * nr) == 0:  # balanced pairs (j, k+1-j): equal backward work
        loads = [sum(spb.suffix_layers(j, k, L) for j in o) for o in owned]
        assert max(loads) - min(loads) <= 2


def test_synthetic_data_matches_reference_generator(orc):
    for widths, N, seed in [([3, 4, 4, 4, 1], 24, 5), ([784, 512, 512, 1], 300, 7), ([1, 1], 3, 0)]:
        X, Y, W = spb.gen_chain_mlp(widths, N, seed)
        Xo, Yo, Wo = orc.gen_chain_mlp(widths, N, seed)
        assert (X == Xo.astype(np.float32)).all()
        assert (Y == Yo.astype(np.float32)).all()
        assert all((a == b.astype(np.float32)).all() for a, b in zip(W, Wo))


def test_config_validation():
    with pytest.raises(spb.ArgumentError):
        spb.SpbConfig(k=3, B=7).validate()
    with pytest.raises(spb.ArgumentError):
        spb.SpbConfig(k=0, B=7).validate()
    spb.SpbConfig(k=4, B=512).validate()
