"""K1 work-item order, restated in Python (CPU): the L2-aware banded order must be a bijection onto
(sequence, q block, head group) and keep the longest band first.  Mirrors of
csrc/prefill_sm100.cuh: prefill_decode_item (band > 0) and prefill_schedule_banded_kernel; the GPU
side of the same logic is covered by tests/test_gpu_parity.py::test_prefill_banded_order_forced."""
import itertools

import pytest


def decode_single(w, nqb, band, num_hg, hpk, useqs=1):
    """prefill_decode_item for a uniform batch (`useqs` sequences of nqb q blocks; analytic).
    band > 0: bands from the top q block down, inside a band by sequence, kv head, q block
    descending; band == 0: q block descending, sequences minor."""
    if band == 0:
        pair, hg = divmod(w, num_hg)
        r, seq = divmod(pair, useqs)
        return seq, nqb - 1 - r, hg
    per_band = band * useqs * num_hg
    i = w // per_band
    r = w - i * per_band
    nq = min(band, nqb - i * band)
    seq, r1 = divmod(r, nq * num_hg)
    per_kvh = nq * hpk
    kvh = r1 // per_kvh
    r2 = r1 - kvh * per_kvh
    e = r2 // hpk
    return seq, nqb - 1 - i * band - e, kvh * hpk + (r2 - e * hpk)


def schedule_banded(lens, causal, hkv, band):
    """prefill_schedule_banded_kernel: entries (seq, q block, kv head), bands descending, inside a
    band by sequence, kv head, q block descending."""
    nqbs = [(n + 127) // 128 for n in lens]
    nbands = (max(nqbs) + band - 1) // band if nqbs and max(nqbs) else 0
    ent = []
    for k in range(nbands - 1, -1, -1):
        for s, nqb in enumerate(nqbs):
            if causal:
                lo, hi = k * band, min(nqb, k * band + band)
            else:
                lo, hi = 0, (nqb if nqb > 0 and (nqb - 1) // band == k else 0)
            for kvh in range(hkv):
                for qb in range(hi - 1, lo - 1, -1):
                    ent.append((s, qb, kvh))
    return ent, sum(nqbs)


def decode_list(w, ent, hpk):
    e = w // hpk
    s, qb, kvh = ent[e]
    return s, qb, kvh * hpk + (w - e * hpk)


@pytest.mark.parametrize("nqb,band,hkv,hpk", [(128, 32, 8, 2), (4, 32, 8, 1), (37, 8, 4, 2), (9, 1, 2, 4), (64, 16, 1, 1)])
def test_single_sequence_banded_decode_is_a_bijection(nqb, band, hkv, hpk):
    num_hg = hkv * hpk
    items = [decode_single(w, nqb, band, num_hg, hpk) for w in range(nqb * num_hg)]
    assert sorted(items) == sorted((0, q, h) for q in range(nqb) for h in range(num_hg))
    # bands are visited top first: the q block never rises by more than a band's span
    first_of_band = [items[i][1] for i in range(0, len(items), band * num_hg)]
    assert first_of_band == sorted(first_of_band, reverse=True)
    # consecutive items of one kv head share its K/V stream: head groups of a kv head are adjacent
    for w in range(0, len(items), hpk):
        assert len({items[w + j][2] // hpk for j in range(hpk)}) == 1


@pytest.mark.parametrize("nqb,band,hkv,hpk,useqs", [(4, 0, 8, 2, 4), (1, 0, 8, 1, 16), (64, 32, 8, 2, 16), (9, 4, 2, 4, 3),
                                                   (37, 0, 4, 2, 5)])
def test_uniform_batch_decode_is_a_bijection(nqb, band, hkv, hpk, useqs):
    """Equal-length batches (no schedule kernel): every (sequence, q block, head group) exactly once,
    longest q blocks first (band 0) or longest band first."""
    num_hg = hkv * hpk
    items = [decode_single(w, nqb, band, num_hg, hpk, useqs) for w in range(nqb * useqs * num_hg)]
    assert sorted(items) == sorted((s, q, h) for s in range(useqs) for q in range(nqb) for h in range(num_hg))
    # bands are anchored at the top q block: band index (nqb - 1 - q) // band never decreases
    key = [nqb - 1 - q if band == 0 else (nqb - 1 - q) // band for _, q, _ in items]
    assert all(a <= b for a, b in itertools.pairwise(key))


@pytest.mark.parametrize("causal", [True, False])
@pytest.mark.parametrize("lens,band", [([300, 77, 1000, 129, 1], 2), ([8192, 128, 4096, 700] * 3, 32), ([0, 5, 0], 1),
                                       ([33430], 32)])
def test_varlen_banded_schedule_is_a_bijection(lens, band, causal):
    hkv, hpk = 8, 2
    ent, n_pairs = schedule_banded(lens, causal, hkv, band)
    assert len(ent) == n_pairs * hkv
    total = n_pairs * hkv * hpk  # = the kernel's total_work = sched[1] * num_hg
    items = [decode_list(w, ent, hpk) for w in range(total)]
    want = [(s, q, h) for s, n in enumerate(lens) for q in range((n + 127) // 128) for h in range(hkv * hpk)]
    assert sorted(items) == sorted(want)
    if causal:  # longest band first: the band index never increases along the list
        bands = [q // band for _, q, _ in items]
        assert all(a >= b for a, b in itertools.pairwise(bands))
