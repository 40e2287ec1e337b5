"""Host-side model of the stream-K schedule of csrc/vlut_kernel_sk.cuh (the
same integer formulas): every (tile, K-tile) unit is processed exactly once,
each CTA produces at most one partial, every owner waits only on CTAs that
produce a partial of the same tile, and the wait graph is acyclic with
producers never waiting -- the deadlock-freedom argument of DESIGN.md."""
import itertools

import pytest


def sk_begin(U, G, c):
    return U * c // G


def sk_seg(u0, u1, KT, j):
    tf, tl = u0 // KT, (u1 - 1) // KT
    kf, kl = u0 % KT, (u1 - 1) % KT + 1
    if tf == tl:
        return tf, kf, kl
    nmid = tl - tf - 1
    if j < nmid:
        return tf + 1 + j, 0, KT
    if j == nmid:
        return tl, 0, kl
    return tf, kf, KT


def sk_nseg(u0, u1, KT):
    return 0 if u1 <= u0 else (u1 - 1) // KT - u0 // KT + 1


def schedule(T, KT, G):
    U = T * KT
    G = min(G, U)
    cover = {}
    produced = {}
    waits = {}
    for c in range(G):
        u0, u1 = sk_begin(U, G, c), sk_begin(U, G, c + 1)
        n = sk_nseg(u0, u1, KT)
        segs = [sk_seg(u0, u1, KT, j) for j in range(n)]
        for tile, ka, kb in segs:
            for kt in range(ka, kb):
                assert (tile, kt) not in cover
                cover[(tile, kt)] = c
        prods = [(t, ka, kb) for t, ka, kb in segs if kb < KT]
        assert len(prods) <= 1
        if prods:
            produced[c] = prods[0]
            # a producer segment precedes any owner segment of the same CTA
            owners = [i for i, (t, ka, kb) in enumerate(segs) if ka > 0 and kb == KT]
            assert all(segs.index(prods[0]) < i for i in owners)
        for t, ka, kb in segs:
            if ka > 0 and kb == KT:  # owner
                head = t * KT
                deps = []
                for c2 in range(c - 1, -1, -1):
                    deps.append(c2)
                    if sk_begin(U, G, c2) <= head:
                        break
                waits[c] = (t, deps)
                # owner processed last in its CTA
                assert segs.index((t, ka, kb)) == n - 1
    assert len(cover) == U
    for c, (t, deps) in waits.items():
        covered = sorted(kt for (tt, kt), cc in cover.items() if tt == t and cc != c)
        for c2 in deps:
            assert c2 in produced and produced[c2][0] == t
            assert c2 not in waits or waits[c2][0] != t
        assert covered == sorted(kt for c2 in deps for kt in range(produced[c2][1], produced[c2][2]))
        # producers never wait before producing: a CTA's producer segment is
        # executed before its owner segment (owner last), so waits point to
        # strictly smaller CTA ids only -> acyclic
        assert all(c2 < c for c2 in deps)
    # K1-32-SK fp32 meeting: a split tile's producers red.add into the slot
    # of its first producer -- the CTA whose range holds the tile's head unit,
    # found by each producer with the owner's walk -- so slots are distinct
    # per tile and every producer and the owner agree on it
    slots = {}
    for c, (t, deps) in waits.items():
        head = t * KT
        slot = min(deps)
        assert sk_begin(U, G, slot) <= head < sk_begin(U, G, slot + 1)
        assert slot not in slots.values()
        slots[t] = slot
    for c, (t, ka, kb) in produced.items():
        head = t * KT
        c_lo = c
        while c_lo > 0 and sk_begin(U, G, c_lo) > head:
            c_lo -= 1
        assert slots[t] == c_lo
    return cover, produced, waits


@pytest.mark.parametrize("T,KT,G", [(72, 40, 148), (160, 160, 148), (1, 1, 148), (5, 3, 148),
                                    (384, 360, 148), (7, 1000, 148), (200, 7, 148), (3, 2, 4)])
def test_streamk_schedule_properties(T, KT, G):
    schedule(T, KT, G)


def test_streamk_schedule_exhaustive_small():
    for T, KT, G in itertools.product(range(1, 9), range(1, 9), range(1, 12)):
        schedule(T, KT, G)
