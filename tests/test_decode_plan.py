"""The engine's decode-attention planner (gpu::Batch::plan_decode via cronus_plan_decode),
host only: every sequence's parts tile its blocks exactly once, parts of a sequence are
contiguous and self-describing (work = seq << 16 | nparts << 8 | part), the list runs
heaviest part first (LPT), and serve-shaped batches (lognormal C2 lengths) are cut so that
no part exceeds the fair share a cluster gets by more than the round-1 rule allowed."""
import numpy as np
import pytest

from paper_2509_17357_b200 import engine as E
from paper_2509_17357_b200.serving import plan_decode


def check_plan(lens, nkv, slots):
    work, item0, C = plan_decode(lens, nkv, slots)
    assert C in (1, 2, 4, 8, 16)
    seq, nparts, part = work >> 16, (work >> 8) & 0xFF, work & 0xFF
    bpp_prev = None
    seen = set()
    for s, n in enumerate(lens):
        i0 = int(item0[s])
        k = int(nparts[i0])
        assert k >= 1
        assert list(seq[i0:i0 + k]) == [s] * k and list(part[i0:i0 + k]) == list(range(k))
        assert all(int(x) == k for x in nparts[i0:i0 + k])
        seen.update(range(i0, i0 + k))
        nblk = (n + 15) // 16
        bpp = -(-nblk // k)
        assert (k - 1) * bpp < nblk  # every part non-empty, parts cover the blocks
    assert seen == set(range(len(work)))
    # LPT: blocks per part non-increasing along the list
    bpps = [-(-((lens[int(s)] + 15) // 16) // int(k)) for s, k in zip(seq, nparts)]
    assert all(a >= b for a, b in zip(bpps, bpps[1:]))
    return work, item0, C


@pytest.mark.parametrize("n", [1, 3, 8, 32, 97, 200])
def test_plan_decode_trace_lengths(n):
    t = E.synth_trace(1000, 1014, 247, E.ALL_AT_ZERO, 0.0, 1)
    rng = np.random.default_rng(n)
    idx = rng.choice(1000, n, replace=False)
    lens = (t.input_len[idx] + (rng.random(n) * t.output_len[idx]).astype(np.int64)).astype(np.int32)
    for slots in (216, 324, 444):
        work, item0, C = check_plan(lens, 8, slots)
        total = int(((lens + 15) // 16).sum()) * 8
        share = max(8, -(-total // slots))
        nblk = (lens + 15) // 16
        nparts = (work >> 8) & 0xFF
        worst = max(-(-int(nblk[s]) // int(nparts[item0[s]])) for s in range(n))
        ctas = len(work) * 8 * C
        wave = slots // 2 if C == 16 else slots
        # never coarser than round 1, unless the coarser plan is one wave (a second wave of this
        # HBM-bound kernel costs more than the makespan model credits)
        assert worst <= max(2 * share * C, -(-int(nblk.max()) // 255)) or ctas <= wave


def test_plan_decode_edge_cases():
    check_plan(np.array([1], np.int32), 8, 216)
    check_plan(np.array([16, 17, 15, 1], np.int32), 4, 296)
    check_plan(np.array([65536, 3, 70000], np.int32), 8, 216)  # <= 255 parts per sequence
    check_plan(np.full(300, 1024, np.int32), 8, 324)
    with pytest.raises(ValueError):
        plan_decode(np.array([], np.int32), 8, 216)
