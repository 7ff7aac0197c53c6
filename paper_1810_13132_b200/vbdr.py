"""Thin Python binding of libvbdr.so (include/vbdr.h) -- argument marshalling only.

PyTorch provides device memory, streams and process groups; every step of the
VBDR path runs in the library's CUDA kernels.  There is no CPU fallback: if the
native library is missing or CUDA is unavailable, construction raises.

Names follow the C ABI: ``vbdr_create`` -> :class:`VBDR`, ``vbdr_scan_slice``
-> :meth:`VBDR.scan_slice`, ``vbdr_slide`` -> :meth:`VBDR.slide`,
``vbdr_estimate`` -> :meth:`VBDR.estimate`, ``vbdr_destroy`` -> :meth:`VBDR.close`.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libvbdr.so")  # the in-tree build

LAYOUT_FAST, LAYOUT_PACKED, LAYOUT_STAMPS = 0, 1, 2
LAYOUTS = {"fast": LAYOUT_FAST, "packed": LAYOUT_PACKED, "stamps": LAYOUT_STAMPS}
ESTIMATORS = {"hll": 0, "loglog": 1, "pcsa": 2}

STATUS = {0: "ok", -1: "EINVAL", -2: "ERANGE", -3: "ESTATE", -4: "ENOMEM", -5: "ECUDA"}


class vbdr_config(C.Structure):
    _fields_ = [("m", C.c_uint32), ("k", C.c_uint32), ("n_phys", C.c_uint64),
                ("seed_a0", C.c_uint32), ("seed_a1", C.c_uint32), ("zbits", C.c_uint32),
                ("rank_cap", C.c_uint32), ("layout", C.c_uint32), ("scan_mode", C.c_uint32),
                ("est_lanes", C.c_uint32), ("est_pass_log2", C.c_uint32),
                ("estimator", C.c_uint32), ("drv_shards", C.c_uint32), ("drv_shard", C.c_uint32)]


class vbdr_info_t(C.Structure):
    _fields_ = [("b", C.c_uint32), ("L", C.c_uint32), ("zbits", C.c_uint32),
                ("fields", C.c_uint32), ("words", C.c_uint32), ("tick", C.c_uint32),
                ("n_phys", C.c_uint64), ("slices_closed", C.c_uint64), ("off_acc", C.c_uint64),
                ("off_sr", C.c_uint64), ("off_drv", C.c_uint64), ("off_regmax", C.c_uint64),
                ("state_bytes", C.c_uint64), ("launches", C.c_uint64),
                ("off_regmax_next", C.c_uint64)]


# Every symbol include/vbdr.h declares (tests check the library exports them).
SYMBOLS = ("vbdr_state_bytes", "vbdr_create", "vbdr_destroy", "vbdr_scan_slice", "vbdr_slide",
           "vbdr_estimate", "vbdr_host_sums", "vbdr_scan_slice_host", "vbdr_estimate_host",
           "vbdr_info", "vbdr_export_ages", "vbdr_export_ages_at", "vbdr_export_regmax",
           "vbdr_export_pool_sums", "vbdr_stamp_delta", "vbdr_slide_delta", "vbdr_debug_set_tick",
           "vbdr_slide_peers", "vbdr_plan_bytes", "vbdr_plan_build", "vbdr_estimate_plan",
           "vbdr_host_sums_plan", "vbdr_plan_check", "vbdr_plan_release",
           "vbdr_estimate_plan_host", "vbdr_config_check", "vbdr_select_above",
           "vbdr_sparse_extract", "vbdr_sparse_apply", "vbdr_last_error", "vbdr_status_string",
           "vbdr_plan_bytes_kind", "vbdr_plan_build_kind", "vbdr_slide_multicast",
           "vbdr_mc_alloc", "vbdr_mc_free", "vbdr_mc_last_error")
PLAN_KINDS = {"auto": 0, "staged": 1, "passid": 2, "sorted": 3}

_lib = None


def lib():
    """Load libvbdr.so (raises if it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: run __graft_entry__.build(); "
                               "there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        vp, u64, u32 = C.c_void_p, C.c_uint64, C.c_uint32
        sig = {
            "vbdr_state_bytes": [C.POINTER(vbdr_config), C.POINTER(u64)],
            "vbdr_create": [C.POINTER(vbdr_config), vp, u64, vp, C.POINTER(vp)],
            "vbdr_destroy": [vp],
            "vbdr_scan_slice": [vp, vp, u64, vp],
            "vbdr_slide": [vp, vp],
            "vbdr_estimate": [vp, vp, u64, vp, vp],
            "vbdr_host_sums": [vp, vp, u64, vp, vp, vp],
            "vbdr_scan_slice_host": [vp, vp, u64, vp, u64, vp],
            "vbdr_estimate_host": [vp, vp, u64, vp, vp, vp, vp],
            "vbdr_info": [vp, C.POINTER(vbdr_info_t)],
            "vbdr_export_ages": [vp, vp, C.c_int, vp],
            "vbdr_stamp_delta": [vp, vp, vp],
            "vbdr_sparse_extract": [vp, u32, vp, u64, vp, vp],
            "vbdr_sparse_apply": [vp, vp, u64, vp, vp],
            "vbdr_debug_set_tick": [vp, u32],
            "vbdr_slide_peers": [vp, vp, u32, u64, u64, vp, vp, vp],
            "vbdr_slide_multicast": [vp, vp, u64, u64, vp],
            "vbdr_mc_alloc": [u64, C.POINTER(vp), C.POINTER(vp), C.POINTER(u64)],
            "vbdr_mc_free": [vp],
            "vbdr_plan_bytes": [vp, u64, C.POINTER(u64)],
            "vbdr_plan_build": [vp, vp, u64, vp, u64, vp],
            "vbdr_plan_bytes_kind": [vp, u64, u32, C.POINTER(u64)],
            "vbdr_plan_build_kind": [vp, vp, u64, u32, vp, u64, vp],
            "vbdr_estimate_plan": [vp, vp, vp, vp],
            "vbdr_host_sums_plan": [vp, vp, vp, vp, vp],
            "vbdr_estimate_plan_host": [vp, vp, vp, vp, vp],
            "vbdr_select_above": [vp, vp, u64, C.c_double, vp, vp, vp],
            "vbdr_plan_check": [vp, vp, vp],
            "vbdr_plan_release": [vp, vp],
            "vbdr_slide_delta": [vp, vp, u64, u64, vp],
            "vbdr_export_ages_at": [vp, vp, u64, vp, vp, C.c_int, vp],
            "vbdr_export_regmax": [vp, vp, vp],
            "vbdr_export_pool_sums": [vp, C.POINTER(u64), C.POINTER(u64), vp],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.vbdr_last_error.argtypes = [vp]
        L.vbdr_last_error.restype = C.c_char_p
        L.vbdr_config_check.argtypes = [C.POINTER(vbdr_config)]
        L.vbdr_config_check.restype = C.c_char_p
        L.vbdr_mc_last_error.argtypes = []
        L.vbdr_mc_last_error.restype = C.c_char_p
        L.vbdr_status_string.argtypes = [C.c_int]
        L.vbdr_status_string.restype = C.c_char_p
        _lib = L
    return _lib


def make_config(m: int, k: int, n_phys: int, seed_a0: int = 0x5EED0001,
                seed_a1: int = 0x5EED0002, zbits: int = 0, rank_cap: int = 0,
                layout: str | int = "fast", scan_mode: int = 0,
                est_lanes: int = 0, est_pass_log2: int = 0,
                estimator: str | int = "hll", drv_shards: int = 0,
                drv_shard: int = 0) -> vbdr_config:
    lay = LAYOUTS[layout] if isinstance(layout, str) else int(layout)
    est = ESTIMATORS[estimator] if isinstance(estimator, str) else int(estimator)
    return vbdr_config(m, k, n_phys, seed_a0, seed_a1, zbits, rank_cap, lay, scan_mode, est_lanes,
                       est_pass_log2, est, drv_shards, drv_shard)


def state_bytes(cfg: vbdr_config) -> int:
    out = C.c_uint64()
    rc = lib().vbdr_state_bytes(C.byref(cfg), C.byref(out))
    if rc != 0:
        why = lib().vbdr_config_check(C.byref(cfg))
        raise ValueError(f"invalid VBDR config: {why.decode() if why else STATUS.get(rc, rc)}")
    return out.value


def _stream_ptr(stream) -> C.c_void_p:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


class VBDR:
    """One VBDR pool on one GPU (``vbdr_create``).  The state tensor is owned here
    (PyTorch memory); the library keeps only pointers into it."""

    def __init__(self, m: int, k: int, n_phys: int, *, seed_a0: int = 0x5EED0001,
                 seed_a1: int = 0x5EED0002, zbits: int = 0, rank_cap: int = 0,
                 layout: str = "fast", scan_mode: int = 0, est_lanes: int = 0,
                 est_pass_log2: int = 0, estimator: str = "hll", device=None, stream=None,
                 state=None, drv_shards: int = 0, drv_shard: int = 0):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("VBDR needs a CUDA device (no CPU fallback)")
        self.device = torch.device(device if device is not None else "cuda")
        self.cfg = make_config(m, k, n_phys, seed_a0, seed_a1, zbits, rank_cap, layout, scan_mode,
                               est_lanes, est_pass_log2, estimator, drv_shards, drv_shard)
        self.estimator = estimator
        nbytes = state_bytes(self.cfg)
        with torch.cuda.device(self.device):
            if state is None:
                state = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            # caller-provided state (e.g. symmetric memory for peer access)
            assert state.dtype == torch.uint8 and state.numel() >= nbytes and state.is_cuda
            self.state = state
            h = C.c_void_p()
            self._check(lib().vbdr_create(C.byref(self.cfg), C.c_void_p(self.state.data_ptr()),
                                          nbytes, _stream_ptr(stream), C.byref(h)), "vbdr_create")
        self._h = h
        self.m, self.k, self.n_phys = m, k, n_phys
        self.layout = layout

    # -------------------------------------------------------------- helpers
    def _check(self, rc: int, what: str):
        if rc != 0:
            h = getattr(self, "_h", None)
            msg = lib().vbdr_last_error(h).decode() if h else ""
            raise RuntimeError(f"{what} failed: {STATUS.get(rc, rc)} {msg}")

    def close(self):
        """``vbdr_destroy`` (the state tensor is released by PyTorch)."""
        if getattr(self, "_h", None):
            lib().vbdr_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        inf = vbdr_info_t()
        self._check(lib().vbdr_info(self._h, C.byref(inf)), "vbdr_info")
        return {name: getattr(inf, name) for name, _ in vbdr_info_t._fields_}

    def sr_view(self):
        """The stamp words as an int32 tensor view for the multi-GPU max merge
        (layout fast: one per BDR; layout stamps: L planes of one per BDR):
        all stamps are < 2^31, so signed MAX is exact."""
        import torch
        inf = self.info()
        if self.layout == "stamps":
            off, n = inf["off_drv"], 4 * inf["words"] * self.n_phys
        elif self.layout == "fast":
            off, n = inf["off_sr"], 4 * self.n_phys
        else:
            raise RuntimeError("layout packed has no mergeable stamps (use the NVLS AND merge)")
        return self.state[off:off + n].view(torch.int32)

    def debug_set_tick(self, tick: int):
        """``vbdr_debug_set_tick`` (tests only)."""
        self._check(lib().vbdr_debug_set_tick(self._h, tick), "vbdr_debug_set_tick")

    def regmax_view(self):
        """The register values M[j] of the last boundary (uint8[n_phys] view)."""
        off = self.info()["off_regmax"]
        return self.state[off:off + self.n_phys]

    def acc_view(self):
        """(S_tot, V_tot) of the last closed slice as an int64[2] view."""
        import torch
        inf = self.info()
        off = inf["off_acc"] + 16 * ((inf["tick"] - 1) & 3)
        return self.state[off:off + 16].view(torch.int64)

    # --------------------------------------------------------------- the path
    def scan_slice(self, pairs, stream=None):
        """``vbdr_scan_slice``: pairs is a device uint32/int32 tensor of 2*n (aip, bip)."""
        assert pairs.is_cuda and pairs.is_contiguous() and pairs.element_size() == 4
        self._check(lib().vbdr_scan_slice(self._h, C.c_void_p(pairs.data_ptr()), pairs.numel() // 2,
                                          _stream_ptr(stream)), "vbdr_scan_slice")

    def slide(self, stream=None, group=None):
        """``vbdr_slide``; with a process group of size > 1, first merge the
        stamp arrays of all ranks by elementwise max (NCCL allreduce MAX)."""
        if group is not None:
            merge_stamps(self, group)
        self._check(lib().vbdr_slide(self._h, _stream_ptr(stream)), "vbdr_slide")

    def stamp_delta(self, out=None, stream=None):
        """``vbdr_stamp_delta``: this slice's max rank per BDR as uint8[n_phys]."""
        import torch
        if out is None:
            out = torch.empty(self.n_phys, dtype=torch.uint8, device=self.device)
        self._check(lib().vbdr_stamp_delta(self._h, C.c_void_p(out.data_ptr()),
                                           _stream_ptr(stream)), "vbdr_stamp_delta")
        return out

    def sparse_extract(self, n_owners: int, cap: int | None = None, stream=None):
        """``vbdr_sparse_extract``: the BDRs this slice touched, as u32 records
        per owner shard.  Returns (records int32[n_owners, cap], counts
        int64[n_owners]); with cap None the exact per-owner counts are taken
        first (one extra pass over the stamps) and cap is their maximum."""
        import torch
        counts = torch.empty(n_owners, dtype=torch.int64, device=self.device)
        if cap is None:
            self._check(lib().vbdr_sparse_extract(self._h, n_owners, None, 0,
                                                  C.c_void_p(counts.data_ptr()),
                                                  _stream_ptr(stream)), "vbdr_sparse_extract")
            cap = max(1, int(counts.max()))
        records = torch.empty((n_owners, cap), dtype=torch.int32, device=self.device)
        self._check(lib().vbdr_sparse_extract(self._h, n_owners, C.c_void_p(records.data_ptr()),
                                              cap, C.c_void_p(counts.data_ptr()),
                                              _stream_ptr(stream)), "vbdr_sparse_extract")
        if int(counts.max()) > cap:
            raise RuntimeError("vbdr_sparse_extract: cap too small")
        return records, counts

    def sparse_extract_into(self, records, counts, stream=None):
        """``vbdr_sparse_extract`` into caller buffers, no host read: records
        int32[n_owners, cap] (slots past an owner's count are left as they
        were), counts int64[n_owners] (the exact totals, possibly > cap)."""
        n_owners, cap = records.shape
        assert records.is_contiguous() and counts.numel() == n_owners
        self._check(lib().vbdr_sparse_extract(self._h, n_owners, C.c_void_p(records.data_ptr()),
                                              cap, C.c_void_p(counts.data_ptr()),
                                              _stream_ptr(stream)), "vbdr_sparse_extract")

    def sparse_apply(self, records, delta_shard, stream=None):
        """``vbdr_sparse_apply``: per-byte max of received records into a shard."""
        self._check(lib().vbdr_sparse_apply(self._h, C.c_void_p(records.data_ptr()),
                                            records.numel(), C.c_void_p(delta_shard.data_ptr()),
                                            _stream_ptr(stream)), "vbdr_sparse_apply")

    def slide_multicast(self, mc_state: int, j0: int = 0, j1: int | None = None, stream=None):
        """``vbdr_slide_multicast``: fused NVLS merge + slide of BDRs [j0, j1);
        mc_state is the multicast address of every rank's state buffer."""
        j1 = self.n_phys if j1 is None else j1
        self._check(lib().vbdr_slide_multicast(self._h, C.c_void_p(mc_state), j0, j1,
                                               _stream_ptr(stream)), "vbdr_slide_multicast")

    def slide_delta(self, delta, j0: int = 0, j1: int | None = None, stream=None):
        """``vbdr_slide_delta``: close the slice from a merged delta over [j0, j1)."""
        j1 = self.n_phys if j1 is None else j1
        assert delta.is_cuda and delta.numel() >= j1 - j0
        self._check(lib().vbdr_slide_delta(self._h, C.c_void_p(delta.data_ptr()), j0, j1,
                                           _stream_ptr(stream)), "vbdr_slide_delta")

    def slide_peers(self, peer_delta, j0: int, j1: int, peer_regmax=None, peer_acc=None,
                    stream=None):
        """``vbdr_slide_peers``: fused merge + slide.  Each list holds one device
        pointer (int) per rank, own rank included (see include/vbdr.h)."""
        n = len(peer_delta)
        arr = lambda xs: (C.c_void_p * n)(*[C.c_void_p(int(x)) for x in xs])  # noqa: E731
        self._check(lib().vbdr_slide_peers(self._h, arr(peer_delta), n, j0, j1,
                                           arr(peer_regmax) if peer_regmax is not None else None,
                                           arr(peer_acc) if peer_acc is not None else None,
                                           _stream_ptr(stream)), "vbdr_slide_peers")

    def acc_ptr(self) -> int:
        """Device address of the accumulator block (vbdr_info off_acc)."""
        return self.state.data_ptr() + self.info()["off_acc"]

    def regmax_ptr(self, next: bool = False) -> int:
        """Device address of the closed tick's register buffer, or with
        next=True of the buffer the next slide writes (the two alternate)."""
        return self.state.data_ptr() + self.info()["off_regmax_next" if next else "off_regmax"]

    def estimate(self, hosts, out=None, stream=None):
        """``vbdr_estimate``: hosts is a device uint32/int32 tensor; returns float64."""
        import torch
        assert hosts.is_cuda and hosts.is_contiguous() and hosts.element_size() == 4
        if out is None:
            out = torch.empty(hosts.numel(), dtype=torch.float64, device=hosts.device)
        self._check(lib().vbdr_estimate(self._h, C.c_void_p(hosts.data_ptr()), hosts.numel(),
                                        C.c_void_p(out.data_ptr()), _stream_ptr(stream)),
                    "vbdr_estimate")
        return out

    def query_top(self, hosts, threshold: float, plan: "EstimatePlan" = None, stream=None):
        """Hosts whose estimate reaches ``threshold``, sorted by estimate
        (descending), ties by ascending host id: the
        estimate (``vbdr_estimate`` or ``vbdr_estimate_plan``) and the
        selection (``vbdr_select_above``) run on the GPU; the short selected
        list is sorted with torch.  Returns (aip uint32 numpy, estimate float64
        numpy)."""
        import numpy as np
        import torch
        est = self.estimate_plan(plan, stream=stream) if plan is not None else \
            self.estimate(hosts, stream=stream)
        n = est.numel()
        idx = torch.empty(max(n, 1), dtype=torch.int32, device=self.device)
        cnt = torch.zeros(1, dtype=torch.int64, device=self.device)
        self._check(lib().vbdr_select_above(self._h, C.c_void_p(est.data_ptr()), n, float(threshold),
                                            C.c_void_p(idx.data_ptr()), C.c_void_p(cnt.data_ptr()),
                                            _stream_ptr(stream)), "vbdr_select_above")
        k = int(cnt.item())
        sel = idx[:k].long()
        e = est[sel].cpu().numpy()
        a = hosts[sel].cpu().numpy().view(np.uint32)
        order = np.lexsort((a, -e))
        return a[order], e[order]

    # ---------------------------------------------------- plan-based estimate
    def plan(self, hosts, kind: str = "auto", stream=None):
        """``vbdr_plan_bytes_kind`` + ``vbdr_plan_build_kind``: preprocess a
        fixed host list (device u32/int32 tensor) for repeated estimates --
        kind "sorted", "staged", "passid" or "auto" (staged for dense host
        lists, else the first that fits; include/vbdr.h vbdr_plan_kind).  Returns an :class:`EstimatePlan`; raises
        ValueError when the pool or host count has no plan of that kind (use
        :meth:`estimate`)."""
        import torch
        n = hosts.numel()
        k = PLAN_KINDS[kind]
        nbytes = C.c_uint64()
        rc = lib().vbdr_plan_bytes_kind(self._h, n, k, C.byref(nbytes))
        if rc != 0:
            raise ValueError(f"no {kind} estimate plan for n_phys={self.n_phys}, {n} hosts")
        buf = torch.empty(nbytes.value, dtype=torch.uint8, device=self.device)
        rc = lib().vbdr_plan_build_kind(self._h, C.c_void_p(hosts.data_ptr()), n, k,
                                        C.c_void_p(buf.data_ptr()), nbytes.value,
                                        _stream_ptr(stream))
        if rc == -2:  # ERANGE: e.g. a block overflows the shared-memory stage
            raise ValueError(lib().vbdr_last_error(self._h).decode())
        self._check(rc, "vbdr_plan_build_kind")
        return EstimatePlan(self, buf, n, kind)

    def estimate_plan(self, plan: "EstimatePlan", out=None, stream=None):
        """``vbdr_estimate_plan``: estimates for the plan's hosts (float64)."""
        import torch
        plan.check_live()
        if out is None:
            out = torch.empty(plan.n_hosts, dtype=torch.float64, device=self.device)
        self._check(lib().vbdr_estimate_plan(self._h, C.c_void_p(plan.buf.data_ptr()),
                                             C.c_void_p(out.data_ptr()), _stream_ptr(stream)),
                    "vbdr_estimate_plan")
        return out

    def estimate_plan_host(self, plan: "EstimatePlan", d_out_stage, h_out, stream=None):
        """``vbdr_estimate_plan_host``: estimates copied into a (pinned) CPU tensor."""
        plan.check_live()
        self._check(lib().vbdr_estimate_plan_host(self._h, C.c_void_p(plan.buf.data_ptr()),
                                                  C.c_void_p(d_out_stage.data_ptr()),
                                                  C.c_void_p(h_out.data_ptr()),
                                                  _stream_ptr(stream)), "vbdr_estimate_plan_host")

    def host_sums_plan(self, plan: "EstimatePlan", stream=None):
        import torch
        plan.check_live()
        S = torch.empty(plan.n_hosts, dtype=torch.int64, device=self.device)
        V = torch.empty(plan.n_hosts, dtype=torch.int32, device=self.device)
        self._check(lib().vbdr_host_sums_plan(self._h, C.c_void_p(plan.buf.data_ptr()),
                                              C.c_void_p(S.data_ptr()), C.c_void_p(V.data_ptr()),
                                              _stream_ptr(stream)), "vbdr_host_sums_plan")
        return S, V

    def plan_check(self, plan: "EstimatePlan", stream=None):
        plan.check_live()
        self._check(lib().vbdr_plan_check(self._h, C.c_void_p(plan.buf.data_ptr()),
                                          _stream_ptr(stream)), "vbdr_plan_check")

    def host_sums(self, hosts, stream=None):
        """``vbdr_host_sums``: per host (S, V) of the integer stage."""
        import torch
        n = hosts.numel()
        S = torch.empty(n, dtype=torch.int64, device=hosts.device)
        V = torch.empty(n, dtype=torch.int32, device=hosts.device)
        self._check(lib().vbdr_host_sums(self._h, C.c_void_p(hosts.data_ptr()), n,
                                         C.c_void_p(S.data_ptr()), C.c_void_p(V.data_ptr()),
                                         _stream_ptr(stream)), "vbdr_host_sums")
        return S, V

    # ---------------------------------------------------- host-buffer path
    def scan_slice_host(self, h_pairs, d_stage, stream=None):
        """``vbdr_scan_slice_host``: h_pairs a (pinned) CPU tensor of 2*n u32."""
        assert not h_pairs.is_cuda and h_pairs.is_contiguous()
        self._check(lib().vbdr_scan_slice_host(self._h, C.c_void_p(h_pairs.data_ptr()),
                                               h_pairs.numel() // 2,
                                               C.c_void_p(d_stage.data_ptr()),
                                               d_stage.numel() // 2, _stream_ptr(stream)),
                    "vbdr_scan_slice_host")

    def estimate_host(self, h_hosts, d_hosts_stage, d_out_stage, h_out, stream=None):
        """``vbdr_estimate_host``: CPU hosts in, CPU float64 estimates out."""
        self._check(lib().vbdr_estimate_host(self._h, C.c_void_p(h_hosts.data_ptr()),
                                             h_hosts.numel(),
                                             C.c_void_p(d_hosts_stage.data_ptr()),
                                             C.c_void_p(d_out_stage.data_ptr()),
                                             C.c_void_p(h_out.data_ptr()), _stream_ptr(stream)),
                    "vbdr_estimate_host")

    # --------------------------------------------------------------- exports
    def export_ages(self, canonical: bool = False, stream=None):
        import numpy as np
        L = self.info()["L"]
        out = np.empty(self.n_phys * L, dtype=np.uint16)
        self._check(lib().vbdr_export_ages(self._h, out.ctypes.data_as(C.c_void_p),
                                           1 if canonical else 0, _stream_ptr(stream)),
                    "vbdr_export_ages")
        return out.reshape(self.n_phys, L)

    def export_ages_at(self, idx, canonical: bool = False, stream=None):
        """``vbdr_export_ages_at``: ages of the sampled BDRs ``idx`` (numpy int)."""
        import numpy as np
        import torch
        inf = self.info()
        d_idx = torch.from_numpy(np.ascontiguousarray(idx, dtype=np.int64)).to(self.device)
        scratch = torch.empty(len(idx) * inf["words"], dtype=torch.int32, device=self.device)
        out = np.empty(len(idx) * inf["L"], dtype=np.uint16)
        self._check(lib().vbdr_export_ages_at(self._h, C.c_void_p(d_idx.data_ptr()), len(idx),
                                              C.c_void_p(scratch.data_ptr()),
                                              out.ctypes.data_as(C.c_void_p),
                                              1 if canonical else 0, _stream_ptr(stream)),
                    "vbdr_export_ages_at")
        return out.reshape(len(idx), inf["L"])

    def export_regmax(self, stream=None):
        import numpy as np
        out = np.empty(self.n_phys, dtype=np.uint8)
        self._check(lib().vbdr_export_regmax(self._h, out.ctypes.data_as(C.c_void_p),
                                             _stream_ptr(stream)), "vbdr_export_regmax")
        return out

    def export_pool_sums(self, stream=None):
        S, V = C.c_uint64(), C.c_uint64()
        self._check(lib().vbdr_export_pool_sums(self._h, C.byref(S), C.byref(V),
                                                _stream_ptr(stream)), "vbdr_export_pool_sums")
        return S.value, V.value


class EstimatePlan:
    """A host list preprocessed by ``vbdr_plan_build`` (device buffer owned here)."""

    def __init__(self, pool: VBDR, buf, n_hosts: int, kind: str = "auto"):
        self.pool, self.buf, self.n_hosts, self.kind = pool, buf, n_hosts, kind

    @property
    def nbytes(self) -> int:
        return self.buf.numel()

    def check_live(self):
        if self.buf is None:
            raise ValueError("this estimate plan was released")

    def release(self):
        if self.buf is not None and getattr(self.pool, "_h", None):
            lib().vbdr_plan_release(self.pool._h, C.c_void_p(self.buf.data_ptr()))
        self.buf = None


class McBuffer:
    """``vbdr_mc_alloc``: device memory bound to a one-device multicast object
    (one GPU: the multicast slide's test path).  ``tensor`` is a uint8 view of
    the unicast mapping (pass it as ``VBDR(state=...)``), ``mc`` the multicast
    address of the same bytes.  Raises RuntimeError without multicast support."""

    class _Iface:
        def __init__(self, ptr, n):
            self.__cuda_array_interface__ = {"shape": (n,), "typestr": "|u1",
                                             "data": (ptr, False), "version": 3}

    def __init__(self, nbytes: int, device=None):
        import torch
        uc, mc, got = C.c_void_p(), C.c_void_p(), C.c_uint64()
        with torch.cuda.device(device if device is not None else torch.cuda.current_device()):
            rc = lib().vbdr_mc_alloc(nbytes, C.byref(uc), C.byref(mc), C.byref(got))
        if rc != 0:
            raise RuntimeError(f"vbdr_mc_alloc failed: {STATUS.get(rc, rc)}: "
                               f"{lib().vbdr_mc_last_error().decode()}")
        self.uc, self.mc, self.nbytes = uc.value, mc.value, got.value
        self.tensor = torch.as_tensor(McBuffer._Iface(self.uc, self.nbytes),
                                      device=torch.device("cuda", torch.cuda.current_device()))

    def free(self):
        if self.uc:
            self.tensor = None
            lib().vbdr_mc_free(C.c_void_p(self.uc))
            self.uc = None


class NvlsMerge:
    """Fused NVLS merge + slide (``vbdr_slide_multicast``) for
    both layouts.  Every rank's pool state lives in torch symmetric memory
    bound to one multicast object; each rank closes its BDR shard with one
    kernel whose loads are reduced by the NVSwitch (MAX of stamps, or AND of
    packed DRV words) and whose registers, pool sums (and packed DRV words)
    land in every rank.  Two device-side barriers (symmetric-memory signal
    pads, no NCCL call) order it after every rank's scan and before the next
    scan or estimate.  The pool must be created with
    ``state=NvlsMerge.alloc_state(...)``.  With one GPU, ``McBuffer`` gives the
    same kernel a one-device multicast object (tests/test_gpu_parity.py)."""

    @staticmethod
    def alloc_state(cfg, device):
        import torch
        import torch.distributed._symmetric_memory as symm
        return symm.empty(state_bytes(cfg), dtype=torch.uint8, device=device)

    def __init__(self, pool: "VBDR", group=None):
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.pool, self.group = pool, group
        self.world, self.rank = _world(group)
        grp = group if group is not None else dist.group.WORLD
        self.handle = symm.rendezvous(pool.state, grp)
        self.mc = int(self.handle.multicast_ptr)
        if not self.mc:
            raise RuntimeError("no multicast object for this group (NVLS unavailable)")
        n = pool.n_phys // self.world
        if n * self.world != pool.n_phys or n % 4:
            raise ValueError("nvls merge needs n_phys divisible by 4 * world size")
        self.j0, self.j1 = self.rank * n, (self.rank + 1) * n

    def close_slice(self, on_merged=None, on_slid=None):
        self.handle.barrier(channel=0)  # every rank's scan of the slice is done
        if on_merged is not None:
            on_merged()
        self.pool.slide_multicast(self.mc, self.j0, self.j1)
        if on_slid is not None:
            on_slid()
        self.handle.barrier(channel=1)  # every rank's registers and sums have landed


# ------------------------------------------------------------ multi-GPU plumbing
def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) of n units for rank (pairs of a slice, or hosts).
    Shards differ in size by at most one unit; their union is [0, n)."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def merge_stamps_tensor(sr, group=None):
    """Elementwise max of every rank's stamp words, in place (allreduce MAX:
    NCCL over NVLink for device tensors, gloo for host tensors in tests).
    Correct because every replica holds identical pre-slice state and max picks
    the newest tick, then the highest rank -- the serial max of PAPER.md:184 is
    commutative and idempotent, so any split of a slice's pairs over ranks gives
    the same merged stamps."""
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return sr
    dist.all_reduce(sr, op=dist.ReduceOp.MAX, group=group)
    return sr


def merge_stamps(pool: "VBDR", group=None):
    """merge_stamps_tensor on the pool's stamp array (layout fast)."""
    return merge_stamps_tensor(pool.sr_view(), group)


MERGE_MODES = ("stamps", "delta", "sharded", "sparse", "p2p", "nvls")


def _world(group):
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def reduce_scatter_max(full, shard, group=None):
    """shard <- this rank's slice of the elementwise MAX of every rank's `full`
    (NCCL reduce-scatter; all-reduce + copy on backends without it)."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.reduce_scatter_tensor(shard, full, op=dist.ReduceOp.MAX, group=group)
    else:
        world, rank = _world(group)
        dist.all_reduce(full, op=dist.ReduceOp.MAX, group=group)
        n = shard.numel()
        shard.copy_(full[rank * n:(rank + 1) * n])
    return shard


def all_gather_shards(full, group=None):
    """In place: every rank contributes its contiguous shard of `full`."""
    import torch.distributed as dist
    world, rank = _world(group)
    n = full.numel() // world
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(full, full[rank * n:(rank + 1) * n], group=group)
    else:
        parts = list(full.split(n))
        mine = parts[rank].clone()
        dist.all_gather(parts, mine, group=group)
    return full


class PeerMerge:
    """Fused merge + slide over NVLink peer memory (``vbdr_slide_peers``).

    Every rank's u8 delta and pool state live in torch symmetric memory, so
    each rank's slide kernel reads its BDR shard of every peer's delta, merges
    them with a per-byte max, slides the shard, and writes the register shard
    and pool sums straight into every rank -- no reduce-scatter or all-gather
    kernels.  Two stream-ordered barriers (tiny NCCL all-reduces) bracket it.
    The pool must be created with ``state=PeerMerge.alloc_state(...)``.
    Verified on one GPU with virtual peers (tests/test_gpu_parity.py); the
    symmetric-memory rendezvous itself needs a multi-GPU box."""

    @staticmethod
    def alloc_state(cfg, device):
        import torch.distributed._symmetric_memory as symm
        import torch
        return symm.empty(state_bytes(cfg), dtype=torch.uint8, device=device)

    def __init__(self, pool: "VBDR", group=None):
        import torch
        import torch.distributed as dist
        import torch.distributed._symmetric_memory as symm
        self.pool, self.group = pool, group
        self.world, self.rank = _world(group)
        grp = group if group is not None else dist.group.WORLD
        self.delta = symm.empty(pool.n_phys, dtype=torch.uint8, device=pool.device)
        hd = symm.rendezvous(self.delta, grp)
        hs = symm.rendezvous(pool.state, grp)
        self.handle = hd
        inf = pool.info()
        self.peer_delta = [hd.buffer_ptrs[r] for r in range(self.world)]
        self.peer_base = [hs.buffer_ptrs[r] for r in range(self.world)]
        self.peer_acc = [hs.buffer_ptrs[r] + inf["off_acc"] for r in range(self.world)]
        n = pool.n_phys // self.world
        if n * self.world != pool.n_phys or n % 4:
            raise ValueError("p2p merge needs n_phys divisible by 4 * world size")
        self.j0, self.j1 = self.rank * n, (self.rank + 1) * n

    def _barrier(self, channel: int = 0):
        # device-side barrier over the symmetric-memory signal pads: a tiny
        # kernel on the current stream, no NCCL call, no host synchronisation
        self.handle.barrier(channel=channel)

    def peer_regmax_next(self) -> list:
        """Every rank's register buffer that the next slide writes (it
        alternates with the tick, which is the same on every rank)."""
        off = self.pool.info()["off_regmax_next"]
        return [b + off for b in self.peer_base]

    def close_slice(self, on_merged=None, on_slid=None):
        """Stamp delta, barrier, fused merge + slide of this rank's shard
        (writing every rank's registers and sums), barrier.  The optional
        callbacks run after the first barrier and after the slide launch
        (bench.py records its phase events there)."""
        self.pool.stamp_delta(self.delta)
        self._barrier(0)  # every rank's delta is written
        if on_merged is not None:
            on_merged()
        self.pool.slide_peers(self.peer_delta, self.j0, self.j1, self.peer_regmax_next(),
                              self.peer_acc)
        if on_slid is not None:
            on_slid()
        self._barrier(1)  # every rank's register shard and sums have landed


def slide_merged(pool: "VBDR", group=None, mode: str = "sharded", delta=None, shard=None):
    """Close the slice on every rank after each scanned its own share of the
    slice's pairs (pairs shard freely: the record is commutative and
    idempotent).

    stamps : allreduce(MAX) of the u32 stamp arrays, full slide on every rank.
    delta  : allreduce(MAX) of the u8 deltas (4x fewer bytes), full slide.
    sharded: reduce-scatter(MAX) of the u8 deltas; each rank slides only its
             1/N of the BDRs, then all-gathers the registers and all-reduces
             the pool sums (bytes and slide time both /N).
    sparse : as sharded, but the ranks exchange only the BDRs their pairs
             touched (vbdr_sparse_extract, all-to-all of u32 records,
             vbdr_sparse_apply): for pools far sparser than a slice.
    Without an initialised process group this is vbdr_slide; a group of one
    still runs the collectives (the N = 1 point of a scaling run, and the
    NCCL calls' test on a one-GPU box: tests/test_gpu_dist.py)."""
    import torch.distributed as dist
    world, rank = _world(group)
    if not dist.is_available() or not dist.is_initialized():
        pool.slide()
        return
    if mode == "stamps":
        merge_stamps(pool, group)
        pool.slide()
        return
    if mode == "sparse":
        _slide_sparse(pool, group, world, rank, shard)
        return
    delta = pool.stamp_delta(delta)
    if mode == "delta":
        dist.all_reduce(delta, op=dist.ReduceOp.MAX, group=group)
        pool.slide_delta(delta)
        return
    if mode != "sharded":
        raise ValueError(f"merge mode {mode!r} not in {MERGE_MODES}")
    n = pool.n_phys // world
    if n * world != pool.n_phys or n % 4:
        raise ValueError("sharded merge needs n_phys divisible by 4 * world size")
    if shard is None:
        import torch
        shard = torch.empty(n, dtype=torch.uint8, device=delta.device)
    reduce_scatter_max(delta, shard, group)
    pool.slide_delta(shard, rank * n, (rank + 1) * n)
    all_gather_shards(pool.regmax_view(), group)
    dist.all_reduce(pool.acc_view(), op=dist.ReduceOp.SUM, group=group)


class SparseMerge:
    """slide_merged(mode="sparse") without host synchronisation on the slice
    path (SURVEY 8(e) iii).  Each rank lists the BDRs its pairs touched as u32
    records per owner shard (``vbdr_sparse_extract``) into a FIXED-capacity
    buffer ``[world, cap]``; one equal-split all-to-all moves every rank's
    ``cap`` records per owner; unused slots stay zero, and a zero record
    (BDR 0, rank 0) is a no-op of ``vbdr_sparse_apply``'s per-byte max.  The
    owner folds the records into its u8 delta shard, slides it, and the
    registers are all-gathered, the pool sums all-reduced.

    ``cap`` is sized once from the exact counts of the first slice (the only
    host read, before any timed work) with ``headroom``, agreed by MAX over
    the ranks.  Later slices never read counts on the host: a device-side
    running maximum is kept, and :meth:`check` (call it after the timed
    region) raises if any owner ever needed more than ``cap`` records --
    records beyond it would have been dropped."""

    def __init__(self, pool: "VBDR", group=None, cap: int | None = None, headroom: float = 1.25):
        import torch
        self.pool, self.group = pool, group
        self.world, self.rank = _world(group)
        n = pool.n_phys // self.world
        if n * self.world != pool.n_phys or n % 4:
            raise ValueError("sparse merge needs n_phys divisible by 4 * world size")
        self.n, self.cap, self.headroom = n, cap, headroom
        dev = pool.device
        self.shard = torch.empty(n, dtype=torch.uint8, device=dev)
        self.counts = torch.empty(self.world, dtype=torch.int64, device=dev)
        self.max_count = torch.zeros((), dtype=torch.int64, device=dev)
        self.records = self.recv = None
        if cap is not None:
            self._alloc(cap)

    def _alloc(self, cap: int):
        import torch
        self.cap = int(cap)
        dev = self.pool.device
        self.records = torch.zeros((self.world, self.cap), dtype=torch.int32, device=dev)
        self.recv = torch.empty(self.world * self.cap, dtype=torch.int32, device=dev)

    def _size_from_first_slice(self):
        import torch
        import torch.distributed as dist
        lib_ = lib()
        self.pool._check(lib_.vbdr_sparse_extract(self.pool._h, self.world, None, 0,
                                                  C.c_void_p(self.counts.data_ptr()),
                                                  _stream_ptr(None)), "vbdr_sparse_extract")
        want = torch.tensor([int(self.counts.max())], dtype=torch.int64, device=self.pool.device)
        if dist.is_available() and dist.is_initialized():
            dist.all_reduce(want, op=dist.ReduceOp.MAX, group=self.group)
        cap = max(1024, int(int(want) * self.headroom + 1023) // 1024 * 1024)
        self._alloc(cap)

    def close_slice(self):
        import torch
        import torch.distributed as dist
        if self.cap is None:
            self._size_from_first_slice()
        self.records.zero_()  # zero record = (BDR 0, rank 0): a no-op of sparse_apply
        self.pool.sparse_extract_into(self.records, self.counts)
        torch.maximum(self.max_count, self.counts.max(), out=self.max_count)
        _all_to_all(self.recv, self.records.view(-1), None, None, self.group)
        self.shard.zero_()
        self.pool.sparse_apply(self.recv, self.shard)
        self.pool.slide_delta(self.shard, self.rank * self.n, (self.rank + 1) * self.n)
        all_gather_shards(self.pool.regmax_view(), self.group)
        dist.all_reduce(self.pool.acc_view(), op=dist.ReduceOp.SUM, group=self.group)

    def check(self):
        """Host check after the timed region: raises if records were dropped."""
        need = int(self.max_count)
        if self.cap is not None and need > self.cap:
            raise RuntimeError(f"sparse merge overflow: an owner needed {need} records, cap "
                               f"{self.cap} (records were dropped: raise cap or headroom)")
        return need


def _slide_sparse(pool: "VBDR", group, world: int, rank: int, shard=None):
    """slide_merged(mode="sparse") through the pool's SparseMerge (created on
    first use for this group)."""
    sm = getattr(pool, "_sparse_merge", None)
    if sm is None or sm.group is not group:
        sm = SparseMerge(pool, group)
        pool._sparse_merge = sm
    sm.close_slice()


def _all_to_all(out, inp, out_sizes, in_sizes, group=None):
    """all_to_all_single (NCCL on the GPU tensors; through host memory on
    backends without CUDA all-to-all, e.g. gloo in the tests)."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_to_all_single(out, inp, output_split_sizes=out_sizes,
                               input_split_sizes=in_sizes, group=group)
        return out
    o = out.cpu()
    dist.all_to_all_single(o, inp.cpu(), output_split_sizes=out_sizes,
                           input_split_sizes=in_sizes, group=group)
    out.copy_(o)
    return out
