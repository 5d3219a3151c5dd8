"""Concurrency stress of the traversal's lock-free hash sets (trav_core.cuh
table_insert: CAS 0 -> 1, key write, release store of 2; readers acquire)
through the C ABI (vr_trav_claim_sigma, vr_trav_bump_keys).

compute-sanitizer (racecheck) is closed on the GPU pool, so the publication
protocol is checked by construction instead: millions of threads insert a few
thousand keys at once (hundreds of copies per key, random order, tables at
load 0.3 to 0.95 so probe chains are long), and every observable must equal
the sequential semantics -- one slot per distinct key, the key stored in that
slot, the smallest row id as the level's claimant (graph.py:105-109's
first-discovery rule restated for a level), edge counts equal to the number
of bumps (graph.py:115-120), and a full table reported as overflow instead of
a hang."""
import ctypes

import numpy as np
import pytest
import torch

from paper_2405_10050_b200 import _lib
from paper_2405_10050_b200.graph import _Tables

pytestmark = pytest.mark.gpu

DEV = torch.device("cuda", 0)


def _p(t):
    return ctypes.c_void_p(t.data_ptr())


class Tabs:
    """Bare vertex / edge tables for dimension d (capacities powers of two)."""

    def __init__(self, d, vcap, ecap, pairs=False):
        z = lambda n: torch.zeros(n, dtype=torch.int32, device=DEV)  # noqa: E731
        self.d = d
        self.vkeys, self.vstate, self.vval, self.vlevel = z(vcap * (d + 1)), z(vcap), z(vcap), z(vcap)
        self.ekeys, self.estate, self.ecount = z(ecap * d), z(ecap), z(ecap)
        if pairs:  # (state, count) pairs in one array: ecount == estate + 1
            self.epairs = z(2 * ecap)
            self.estate, self.ecount = self.epairs[0::2], self.epairs[1::2]
        self.overflow = z(1)
        self.T = _Tables(_p(self.vkeys).value, _p(self.vstate).value, _p(self.vval).value,
                         _p(self.vlevel).value, vcap, _p(self.ekeys).value, _p(self.estate).value,
                         _p(self.ecount).value, ecap, _p(self.overflow).value)

    def claim(self, rows, level):
        n = rows.shape[0]
        slot = torch.empty(n, dtype=torch.int64, device=DEV)
        newf = torch.empty(n, dtype=torch.int32, device=DEV)
        _lib.check(_lib.lib().vr_trav_claim_sigma(ctypes.byref(self.T), self.d, _p(rows), n, level,
                                                  _p(slot), _p(newf), None), "claim_sigma")
        torch.cuda.synchronize()
        return slot.cpu().numpy(), newf.cpu().numpy()

    def bump(self, keys):
        n = keys.shape[0]
        out = torch.empty(n, dtype=torch.int32, device=DEV)
        _lib.check(_lib.lib().vr_trav_bump_keys(ctypes.byref(self.T), self.d, _p(keys), n,
                                                _p(out), None), "bump_keys")
        torch.cuda.synchronize()
        return out.cpu().numpy()


def _distinct_sorted_rows(rng, k, width, hi):
    rows = set()
    while len(rows) < k:
        rows.add(tuple(sorted(rng.choice(hi, width, replace=False).tolist())))
    return np.array(sorted(rows), dtype=np.int32)


@pytest.mark.parametrize("d,vcap,copies", [(3, 1 << 13, 400), (5, 1 << 13, 400),
                                            (8, 1 << 13, 256), (4, 1 << 12, 600)])
def test_claim_sigma_under_contention(d, vcap, copies):
    rng = np.random.default_rng(d)
    k = int(0.3 * vcap) if vcap >= 1 << 13 else int(0.95 * vcap)  # load 0.3 / 0.95
    keys = _distinct_sorted_rows(rng, k, d + 1, 10 ** 6)
    which = rng.integers(0, k, k * copies)
    which[:k] = np.arange(k)  # every key present
    rng.shuffle(which)
    rows = torch.from_numpy(keys[which]).to(DEV)
    tb = Tabs(d, vcap, 1 << 10)
    slot, newf = tb.claim(rows, level=7)
    assert int(tb.overflow.item()) == 0
    assert (slot >= 0).all()
    # one slot per distinct key, distinct keys in distinct slots
    first_slot = np.full(k, -1, dtype=np.int64)
    first_slot[which] = slot
    assert np.array_equal(slot, first_slot[which]), "a key landed in two slots"
    assert len(np.unique(first_slot)) == k, "two keys share a slot"
    # the stored key is the row's key, the slot is published
    vk = tb.vkeys.view(-1, d + 1).cpu().numpy()
    assert np.array_equal(vk[slot], keys[which])
    assert (tb.vstate.cpu().numpy()[first_slot] == 2).all()
    assert int((tb.vstate.cpu().numpy() == 2).sum()) == k
    # exactly one claimant per key: the smallest row id
    smallest = np.full(k, len(which), dtype=np.int64)
    np.minimum.at(smallest, which, np.arange(len(which)))
    assert int(newf.sum()) == k
    assert np.array_equal(np.nonzero(newf)[0], np.sort(smallest))
    assert np.array_equal(tb.vval.cpu().numpy()[first_slot], smallest)
    # a later level: old keys are found (not new), fresh keys claimed once
    fresh = _distinct_sorted_rows(np.random.default_rng(100 + d), 64, d + 1, 10 ** 6)
    fresh = fresh[~(fresh[:, None, :] == keys[None, :, :]).all(2).any(1)]
    mix = np.concatenate([keys[rng.integers(0, k, 4096)], np.repeat(fresh, 8, 0)])
    rng.shuffle(mix)
    if k + len(fresh) <= vcap:
        slot2, newf2 = tb.claim(torch.from_numpy(np.ascontiguousarray(mix)).to(DEV), level=8)
        assert int(tb.overflow.item()) == 0
        is_old = (mix[:, None, :] == keys[None, :, :]).all(2).any(1)
        assert not newf2[is_old].any()
        assert int(newf2.sum()) == len(fresh)


@pytest.mark.parametrize("pairs", [False, True])
@pytest.mark.parametrize("d,ecap", [(3, 1 << 14), (6, 1 << 14), (8, 1 << 13)])
def test_bump_keys_counts_every_bump(d, ecap, pairs):
    rng = np.random.default_rng(10 + d)
    k = int(0.9 * ecap)  # long probe chains
    keys = _distinct_sorted_rows(rng, k, d, 10 ** 6)
    mult = rng.integers(1, 40, k)
    which = np.repeat(np.arange(k), mult)
    rng.shuffle(which)
    tb = Tabs(d, 1 << 10, ecap, pairs=pairs)
    out = tb.bump(torch.from_numpy(keys[which]).to(DEV))
    assert int(tb.overflow.item()) == 0
    assert np.array_equal(out, mult[which]), "lost or duplicated edge bumps"
    assert int(tb.ecount.sum().item()) == int(mult.sum())
    assert int((tb.estate.cpu().numpy() == 2).sum()) == k


def test_full_table_reports_overflow():
    d = 3
    rng = np.random.default_rng(0)
    keys = _distinct_sorted_rows(rng, 3000, d + 1, 10 ** 5)
    rows = torch.from_numpy(np.repeat(keys, 4, 0)).to(DEV)
    tb = Tabs(d, 1 << 11, 1 << 10)  # 2048 slots for 3000 keys
    slot, _ = tb.claim(rows, level=1)
    assert int(tb.overflow.item()) == 1
    assert (slot < 0).any()
    assert int((tb.vstate.cpu().numpy() == 2).sum()) == 1 << 11
