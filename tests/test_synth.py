"""The shared seeded generator (synth/): determinism and workload shape."""
import numpy as np

import synth


def test_deterministic_and_chunkable():
    tr = synth.CONFIGS["tiny"]
    a = synth.generate(tr, 3)
    b = synth.generate(tr, 3)
    assert a.shape == (10_000, 2) and a.dtype == np.uint32
    assert np.array_equal(a, b)
    # counter-based: any sub-range regenerates identically
    assert np.array_equal(synth.generate(tr, 3, start=1234, count=777), a[1234:2011])
    assert not np.array_equal(synth.generate(tr, 4), a)


def test_hosts_distinct_and_zipf_share():
    tr = synth.CONFIGS["tiny"]
    ids = tr.host_ids()
    assert len(set(ids.tolist())) == tr.hosts
    p = synth.generate(tr, 0)
    assert set(np.unique(p[:, 0]).tolist()) <= set(ids.tolist())
    share = (p[:, 0] == ids[0]).mean()
    w = np.arange(1, 65, dtype=float) ** -1.1
    assert abs(share - w[0] / w.sum()) < 0.02  # ~25 % at H=64


def test_cardinality_structure():
    """Repeated pairs within and across slices; window cardinality between the
    slice cardinality and k times it."""
    tr = synth.CONFIGS["tiny"]
    s = [synth.generate(tr, t) for t in range(4)]
    key = lambda p: set((p[:, 0].astype(np.uint64) << 32 | p[:, 1]).tolist())
    one = len(key(s[0]))
    win = len(set().union(*[key(x) for x in s]))
    assert one < 10_000  # duplicates within a slice
    assert one < win < 4 * one
