"""CPU-side checks of the C ABI library: it loads without a GPU, exports every
symbol include/vbdr.h declares, and validates configurations on the host."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def vb():
    from paper_1810_13132_b200 import _build, vbdr
    _build.build_vbdr()
    return vbdr


def _declared():
    src = open(os.path.join(ROOT, "include", "vbdr.h")).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+char\s*\*|vbdr_status)\s*(vbdr_\w+)\s*\(", src,
                                 re.M)))


def test_header_declares_the_boundary():
    names = _declared()
    for n in ("vbdr_create", "vbdr_scan_slice", "vbdr_slide", "vbdr_estimate", "vbdr_destroy"):
        assert n in names
    assert len(names) == len(set(names)) >= 31


def test_library_exports_every_declared_symbol(vb):
    out = subprocess.run(["nm", "-D", "--defined-only", vb.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (vbdr_\w+)", out))
    for n in _declared():
        assert n in exported, n
    assert set(vb.SYMBOLS) == set(_declared())
    lib = vb.lib()
    for n in _declared():
        getattr(lib, n)


def test_sm100a_code_only(vb):
    out = subprocess.run(["cuobjdump", "--list-elf", vb.LIB_PATH], capture_output=True, text=True,
                         check=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_[0-9]+[^0a-z]", out.replace("sm_100a", ""))


def test_state_bytes_and_validation(vb):
    cfg = vb.make_config(128, 5, 1 << 22, scan_mode=5)
    # layout F: acc 256 B + sr 16 MiB + DRV 3 planes * 16 MiB + two regmax buffers of 4 MiB
    assert vb.state_bytes(cfg) == 256 + 4 * (1 << 22) + 12 * (1 << 22) + 2 * (1 << 22)
    assert vb.state_bytes(vb.make_config(128, 5, 1 << 22)) == vb.state_bytes(cfg)
    assert vb.state_bytes(vb.make_config(128, 5, 1 << 22, scan_mode=2)) == vb.state_bytes(cfg)
    # the measured-slower round-1 scan modes are not in the product library
    for mode in (1, 3, 4, 6, 7):
        with pytest.raises(ValueError, match="scan_mode"):
            vb.state_bytes(vb.make_config(128, 5, 1 << 22, scan_mode=mode))
    cfgp = vb.make_config(128, 5, 1 << 22, layout="packed")
    assert vb.state_bytes(cfgp) == 256 + 12 * (1 << 22) + 2 * (1 << 22)
    # bigwin: zb = 6, F = 5, W = 5
    assert vb.state_bytes(vb.make_config(256, 60, 1 << 28, scan_mode=5)) == \
        256 + (4 + 20 + 2) * (1 << 28)
    assert vb.state_bytes(vb.make_config(256, 60, 1 << 28)) == \
        256 + (4 + 20 + 2) * (1 << 28)
    bad = [dict(m=3, k=5, n_phys=1 << 10), dict(m=512, k=5, n_phys=1 << 9),
           dict(m=32, k=0, n_phys=1 << 12), dict(m=32, k=4, n_phys=3000),
           dict(m=32, k=8, n_phys=1 << 12, zbits=3), dict(m=32, k=4, n_phys=1 << 12, rank_cap=28),
           dict(m=2, k=4, n_phys=1 << 30)]
    for kw in bad:
        with pytest.raises(ValueError, match="invalid VBDR config: "):
            vb.state_bytes(vb.make_config(**kw))
    # a rank cap relaxes the exact-sum bound n_phys * 2^L <= 2^53
    vb.state_bytes(vb.make_config(2, 4, 1 << 30, rank_cap=20))
    # packed layout auto-bumps zb when k = 2^zb - 1 (R#2); explicit zb=3, k=7 is rejected
    vb.state_bytes(vb.make_config(32, 7, 1 << 12, layout="packed"))
    with pytest.raises(ValueError):
        vb.state_bytes(vb.make_config(32, 7, 1 << 12, zbits=3, layout="packed"))


def test_register_sharded_state_bytes_and_validation(vb):
    full = vb.state_bytes(vb.make_config(128, 5, 1 << 22, scan_mode=5))
    sharded = vb.state_bytes(vb.make_config(128, 5, 1 << 22, scan_mode=5, drv_shards=4, drv_shard=3))
    assert full - sharded == 12 * (1 << 22) * 3 // 4  # 3 DRV planes, 3/4 of the BDRs gone
    for kw in (dict(drv_shards=4, drv_shard=4), dict(drv_shards=0, drv_shard=1),
               dict(drv_shards=3), dict(drv_shards=2, layout="packed")):
        with pytest.raises(ValueError, match="invalid VBDR config: "):
            vb.state_bytes(vb.make_config(128, 5, 1 << 22, **kw))


def test_shard_range_partitions():
    from paper_1810_13132_b200 import shard_range
    for n in (0, 1, 7, 100, 5_000_001):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1


def test_binding_refuses_without_cuda(vb):
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError):
        vb.VBDR(32, 4, 1 << 12)
