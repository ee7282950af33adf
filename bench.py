#!/usr/bin/env python3
"""Benchmark of the hot path: exact matching of short patterns (m = 2..32), every position.

Workload (N = 1): BASELINE.json configs[1], the random-alphabet sweep -- n = 256 MiB texts
i.i.d. uniform over byte values 0..sigma-1 for sigma in {2,4,...,256}; for every (sigma, m in
{2,4,8,16,32}) 100 patterns extracted from the text at seeded uniform positions (the paper's
protocol); every search reports all its positions into its own buffer.
One STEP = the whole sweep: 8 texts x 5 m x 100 patterns = 4000 searches, through the public
API: per text, the equality-mask index over the byte values its dense searches read
(epsm_eqidx_build_async, rebuilt every step), then per m ONE group call
(epsm_group_search_index_async): the group's sparse patterns share one pass over the text,
its dense patterns (their positions dominate) are searched one by one over the index.

Metric: text GB/s scanned = 1e9 bytes of text per second, where a search of a 256 MiB text
counts 256 MiB (the paper's and SURVEY 8(d)'s definition).  Every text is larger than the
126 MB L2, so no flush is inserted.  Parity: warm-up step 0 checks every (sigma, m) group
against the ORACLE -- the full-text count of one search per group and the positions of two
searches per group in 1 MiB windows (first, last, random); tests/ hold the full parity suite.

N > 1 (one process per GPU, torchrun; `--gpus N` re-launches itself under torchrun when
WORLD_SIZE is unset): weak scaling -- every rank holds a 256 MiB shard (+31-byte halo) of an
N x 256 MiB text per sigma.  Per group: range group search over the owned starts, NCCL
all-gather of the [N, 100] count matrix, then the positions all-gather (epsm_allgatherv_async:
grouped ncclBroadcasts) so that every rank holds every search's global positions -- the
north_star multi-GPU path.  `--keep-sharded` drops the gather (positions stay on the rank
that found them).  Scan, count-exchange and gather times are reported separately.

--impl reference: the CPU oracle (brute force, oracle/) timed on this box's host cores over a
bounded sample of the same workload (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402

METRIC = "text GB/s scanned (bit-exact positions) vs HBM peak, m=2..32, 1/2/4/8 B200"
UNIT = "GB/s"
SIGMAS = (2, 4, 8, 16, 32, 64, 128, 256)
MS = (2, 4, 8, 16, 32)
N_PER_RANK = 256 * synth.MiB
WINDOW = 1 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="epsm", choices=["epsm", "reference"])
    ap.add_argument("--patterns", type=int, default=100, help="patterns per (sigma, m)")
    ap.add_argument("--sigmas", default=",".join(map(str, SIGMAS)))
    ap.add_argument("--ms", default=",".join(map(str, MS)))
    ap.add_argument("--mode", default="group", choices=["group", "batch"],
                    help="group: epsm_group_search_index_async per (sigma, m) (default); batch: the "
                         "per-search batch API epsm_search_batch_index_async (A/B)")
    ap.add_argument("--keep-sharded", action="store_true", help="N > 1: no positions all-gather")
    ap.add_argument("--gather-budget-gb", type=float, default=24.0,
                    help="N > 1: device bytes for gathered positions (searches gathered in sub-batches)")
    ap.add_argument("--e2e-steps", type=int, default=1)
    ap.add_argument("--e2e-host-gb", type=float, default=40.0, help="pinned host memory for e2e positions")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true")
    ap.add_argument("--no-breakdown", action="store_true")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the `configs` field (BASELINE configs 1, 3a, 3b, 4, 5a, 5b via the group search)")
    ap.add_argument("--scan-patterns", type=int, default=10,
                    help="online scan field: patterns per (sigma, m), one search per launch (0: off)")
    ap.add_argument("--cpu-bytes", type=int, default=64 * synth.MiB, help="host baseline sample bytes per search")
    ap.add_argument("--out", default=None, help="also write the JSON line here")
    return ap.parse_args()


def maybe_relaunch(args):
    """`python bench.py --gpus N` (N > 1) without torchrun: re-exec under torchrun, one rank per GPU."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    os.execv(sys.executable, cmd)


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: copy, read + write)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def roofline_block(achieved, achieved8d, moved, alg8d, hbm_peak, peak_src, tf, gather, kt_n, kt_ms, kt_bytes,
                   steps, ms_step):
    """The line's `roofline`: the dominant kernel (the positions fan-out) timed live with CUDA events on
    its own stream over the timed region -- its algorithmic bytes per launch (source positions read once,
    every output's positions written) over its mean launch duration -- and, under `step`, every kernel
    of the timed region together (bytes the step must move over the step time)."""
    step = {"achieved": round(achieved, 1), "frac": round(achieved / hbm_peak, 4),
            "kernel": "every kernel of the timed region (group passes, single-pattern index/text "
                      "searches, index builds, fan-out copies), one stream, back to back",
            "bytes": "moved: index build n + nv*n/8; per shared group pass the text once; per "
                     "dense distinct pattern d*n/8 planes (index) or n (text), plus its positions "
                     "read once by the fan-out copy when it has duplicates; 8 B per position written"
                     + ("; gathered positions received" if gather else ""),
            "moved_bytes_per_step": int(moved)}
    r = {"bound": "hbm", "peak": hbm_peak, "unit": "GB/s", "peak_source": peak_src}
    kern = (tf or {}).get("kernels") or {}
    if kt_n and kt_ms > 0:
        dom = "epsm_replicate_multi_kernel"
        a = kt_bytes / kt_n / (kt_ms / kt_n * 1e-3) / 1e9
        r.update({"achieved": round(a, 1), "frac": round(a / hbm_peak, 4),
                  "traffic": (kern.get(dom) or {}).get("dram_bytes_per_busy_launch",
                                                       (kern.get(dom) or {}).get("dram_bytes_per_launch")),
                  "kernel": dom + " (the positions fan-out to the searches that share a pattern)",
                  "launches_per_step": round(kt_n / steps, 2),
                  "us_per_launch": round(kt_ms / kt_n * 1e3, 1),
                  "bytes_per_launch": int(kt_bytes / kt_n),
                  "share_of_step_live": round(kt_ms / steps / ms_step, 4),
                  "share_of_step_ncu": (kern.get(dom) or {}).get("share"),
                  "timing": "CUDA events recorded by the library on the kernel's stream around each of its "
                            "launches in the timed region (epsm_ktimer_enable)",
                  "bytes": "per job 8*occ of source positions read once + 8*occ written per output"})
    else:
        r.update({"achieved": step["achieved"], "frac": step["frac"], "traffic": None,
                  "kernel": step["kernel"], "bytes": step["bytes"]})
    r.update({"step": step,
              "survey_8d": {"bytes_per_step": int(alg8d), "achieved": round(achieved8d, 1),
                            "frac": round(achieved8d / hbm_peak, 4),
                            "note": "n + 8*occ per search as SURVEY 8(d) writes it: every search "
                                    "counted as a full text pass, so frac > 1 where searches share "
                                    "one pass or read planes -- not HBM evidence"},
              "traffic_unit": (tf or {}).get("unit"),
              "kernel_shares_ncu": {k: v.get("share") for k, v in kern.items()}})
    return r


def traffic_file():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


# ----------------------------------------------------------------- clocks

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = os.path.join("/tmp", f"epsm_clocks_{os.getpid()}_{index}.csv")

    def __enter__(self):
        try:
            self.f = open(self.path, "w")
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"], stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
            return self
        t0 = time.time()                          # the first sample before the timed region
        while time.time() - t0 < 3.0 and os.path.getsize(self.path) == 0:
            time.sleep(0.02)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.f.close()

    def summary(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        rows = []
        with open(self.path) as f:
            for line in f:
                parts = [x.strip() for x in line.split(",")]
                if len(parts) >= 8:
                    rows.append(parts)
        try:
            os.remove(self.path)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(r[0]) for r in rows) if v is not None]
        mx = [v for v in (num(r[1]) for r in rows) if v is not None]
        pw = [v for v in (num(r[2]) for r in rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "power_w_max": max(pw) if pw else None}


# ----------------------------------------------------------------- distributed

def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test hook: EPSM_BENCH_EMULATE=1 runs every rank on cuda:0 over gloo (a host-side check of
    # the N > 1 logic on a one-GPU box; no kernel waits on another rank, only gloo does)
    emulate = os.environ.get("EPSM_BENCH_EMULATE") == "1"
    if emulate:
        local = 0
    if world > 1:
        import torch.distributed as dist
        if args.impl == "epsm" and not emulate:
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    if args.gpus > 1 and world != args.gpus and rank == 0:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE = {world}", file=sys.stderr)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, world: int, dev) -> float:
    if world == 1:
        return x
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=dev if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------- workload

def make_texts(sigmas, world, rank, dev):
    """Per sigma: (sigma, spec, n_total, base, owned, shard tensor on dev)."""
    from paper_1209_6449_b200 import sharding
    out = []
    n_total = N_PER_RANK * world
    for s in sigmas:
        spec = synth.raw_sigma_spec(s, (2, s))
        base, owned, slen = sharding.shard_layout(n_total, world, rank)
        t = synth.text_torch(spec, base, slen, device=dev)
        out.append((s, spec, n_total, base, owned, t))
    return out


def make_patterns(texts, ms, count):
    pats = {}
    for s, spec, n_total, base, owned, t in texts:
        for m in ms:
            if base == 0 and t.numel() == n_total:
                p, _ = synth.extract_patterns_torch(t, (2, s, m), m, count)
            else:
                p, _ = synth.extract_patterns_spec(spec, n_total, (2, s, m), m, count)
            pats[(s, m)] = p
    return pats


def check_windows(pat: bytes, pos: torch.Tensor, occ: int, spec, n_total: int, rng) -> None:
    """Oracle parity of one search's positions (device tensor, first occ valid, global) in 1 MiB
    windows of the global text: the first, the last and a random one (the text is counter-based,
    so any window is generated on the host independently of the GPU)."""
    import oracle
    m = len(pat)
    w = min(WINDOW, n_total)
    starts = {0, n_total - w, int(rng.integers(0, max(1, n_total - w + 1)))}
    valid = pos[:occ]
    for a in sorted(starts):
        host = synth.text_np(spec, a, w)
        want = oracle.search(pat, host).astype(np.int64) + a
        lo = int(torch.searchsorted(valid, torch.tensor([a], device=pos.device)).item())
        hi = int(torch.searchsorted(valid, torch.tensor([a + w - m + 1], device=pos.device)).item())
        got = valid[lo:hi].cpu().numpy()
        assert np.array_equal(got, want), f"oracle window mismatch: m={m} window {a} ({got[:4]} vs {want[:4]})"


# ----------------------------------------------------------------- GPU arm

def run_epsm(args, world, rank, local):
    import paper_1209_6449_b200 as epsm
    from paper_1209_6449_b200 import sharding
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)
    sigmas = [int(x) for x in args.sigmas.split(",")]
    ms = [int(x) for x in args.ms.split(",")]
    P = args.patterns
    texts = make_texts(sigmas, world, rank, dev)
    pats = make_patterns(texts, ms, P)
    G = []                                       # (text index, m, group, plans or None)
    for ti, (s, *_rest) in enumerate(texts):
        for m in ms:
            g = epsm.group(pats[(s, m)])
            plans = [epsm.plan(p) for p in pats[(s, m)]] if args.mode == "batch" else None
            G.append((ti, m, g, plans))
    # the index of each text: the byte values its dense searches read (group mode), or every
    # qualifying search's values (batch mode)
    ixv, ixs = {}, {}
    for ti in range(len(texts)):
        if args.mode == "group":
            vals = sorted({v for gti, _, g, _ in G if gti == ti for v in g.index_values()})
        else:
            vals = list(epsm.index_values([pl for gti, _, _, pls in G if gti == ti for pl in pls]))
        if vals:
            ixv[ti] = bytes(vals)
            ixs[ti] = epsm.EqIndex()
    occ_loc = torch.zeros((len(G), P), dtype=torch.int64, device=dev)
    occ_glob = torch.zeros((len(G), P), dtype=torch.int64, device=dev) if world > 1 else occ_loc
    gather = world > 1 and not args.keep_sharded
    n_text_step = sum(texts[ti][2] for ti, *_ in G) * P          # global text bytes per step

    def run_group(gi, outs):
        ti, m, g, plans = G[gi]
        s_, spec_, n_total_, base_, owned_, t_ = texts[ti]
        ix = ixs.get(ti)
        if world == 1:
            if plans is None:
                g.search_async(t_, occ_loc[gi], outs=outs, index=ix)
            else:
                epsm.search_batch_async(plans, t_, occ_loc[gi], outs=outs, index=ix)
        else:
            g.search_range_async(t_, owned_, base_, n_total_, occ_loc[gi], outs=outs, index=ix)

    # sizing pass (counts only) -> one output buffer per search of a group (reused by every
    # group; stream order keeps consecutive groups apart)
    for ti in ixs:
        ixs[ti].build_async(texts[ti][5], ixv[ti])
    for gi in range(len(G)):
        run_group(gi, None)
    torch.cuda.synchronize()
    pcap = int(occ_loc.max().item()) + 1
    pool = [torch.empty(pcap, dtype=torch.int64, device=dev) for _ in range(P)]
    gpool, cm_all = [], [None] * len(G)
    if gather:
        cm0 = sharding.exchange_count_matrix(occ_loc.reshape(-1)).view(world, len(G), P)
        gcap = int(cm0.sum(0).max().item()) + 1
        nbuf = int(max(1, min(P, args.gather_budget_gb * 1e9 // (8 * gcap))))
        gpool = [torch.empty(gcap, dtype=torch.int64, device=dev) for _ in range(nbuf)]

    rng = np.random.default_rng(12345 + rank)
    phase = {"scan": 0.0, "counts": 0.0, "gather": 0.0}

    def one_step(check=False, phase_ev=None, group_ev=None):
        last = None
        for gi, (ti, m, g, plans) in enumerate(G):
            if ti != last and ti in ixs:
                if group_ev is not None:
                    group_ev[("ix", ti)] = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                    group_ev[("ix", ti)][0].record(stream)
                ixs[ti].build_async(texts[ti][5], ixv[ti])
                if group_ev is not None:
                    group_ev[("ix", ti)][1].record(stream)
            last = ti
            if group_ev is not None:
                group_ev[gi] = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
                group_ev[gi][0].record(stream)
            if phase_ev is not None:
                e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
                e[0].record(stream)
            run_group(gi, pool)
            if phase_ev is not None:
                e[1].record(stream)
            if world > 1:
                cm = sharding.exchange_count_matrix(occ_loc[gi])
                occ_glob[gi].copy_(cm.sum(0))
                if phase_ev is not None:
                    e[2].record(stream)
                if gather:
                    cmh = cm.cpu().numpy()                     # sizes of the gather (host)
                    cm_all[gi] = cmh
                    for a in range(0, P, len(gpool)):
                        b = min(P, a + len(gpool))
                        sharding.gather_batch_positions(pool[a:b], cmh[:, a:b], gpool[:b - a])
                        if check:
                            torch.cuda.synchronize()
                            for jj in (a, b - 1):
                                check_windows(pats[(texts[ti][0], m)][jj], gpool[jj - a], int(cmh[:, jj].sum()),
                                              texts[ti][1], texts[ti][2], rng)
                elif check:
                    torch.cuda.synchronize()
            elif check:
                torch.cuda.synchronize()
                occ_h = occ_loc[gi].cpu().numpy()
                for jj in (0, P - 1):
                    check_windows(pats[(texts[ti][0], m)][jj], pool[jj], int(occ_h[jj]), texts[ti][1],
                                  texts[ti][2], rng)
            if phase_ev is not None:
                e[3].record(stream)
                phase_ev.append(e)
            if group_ev is not None:
                group_ev[gi][1].record(stream)

    # warm-up; step 0 is also the oracle parity check
    for w in range(args.warmup):
        one_step(check=(w == 0 and not args.no_check))
    torch.cuda.synchronize()
    checked = None
    if not args.no_check:
        checked = oracle_full_counts(args, texts, pats, G, occ_glob, world, rank)

    # timed region: K steps back to back, bracketed by barrier + synchronize and CUDA events
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = epsm.launch_count()
    epsm.ktimer_read()                                   # (drop records of the warm-up)
    epsm.ktimer_enable(True)                             # events around every fan-out launch
    with ClockSampler(local) as clk:
        barrier(world)
        torch.cuda.synchronize()
        start.record(stream)
        for _ in range(args.steps):
            one_step()
        stop.record(stream)
        torch.cuda.synchronize()
        barrier(world)
    launches = epsm.launch_count() - launches0
    epsm.ktimer_enable(False)
    kt_n, kt_ms, kt_bytes = epsm.ktimer_read()           # the dominant kernel, timed live
    ms_total = max_over_ranks(start.elapsed_time(stop), world, dev)
    ms_step = ms_total / args.steps
    value = n_text_step * args.steps / (ms_total * 1e-3) / 1e9
    clocks = clk.summary()

    # bytes per step, two accountings:
    #  * SURVEY 8(d) as written: n + 8 * occ per search (every search counted as a text pass);
    #  * moved: what the kernels must read / write -- per index build n + nv*n/8; per group the
    #    text once per shared pass; per dense search its planes (d*n/8) or the text; 8 per
    #    position written; (N > 1) the gathered positions received from the other ranks
    occ_l = occ_loc.cpu().numpy().astype(np.int64)
    occ_g = occ_glob.cpu().numpy().astype(np.int64)
    moved = 0.0
    rows_moved = {}
    for gi, (ti, m, g, plans) in enumerate(G):
        nb = texts[ti][5].numel()
        b = 8.0 * occ_l[gi].sum()
        if args.mode == "group":
            flags = g.dense_searches()
            info = g.info()
            b += nb * len(info["passes"])
            dense = {}                                   # dense distinct pattern -> its searches
            for j, fl in enumerate(flags):
                if fl:
                    dense.setdefault(pats[(texts[ti][0], m)][j], []).append(j)
            for p, js in dense.items():                  # one scan per distinct dense pattern
                pv = epsm.plan(p)
                iv = pv.index_values()
                pv.close()
                b += nb * len(iv) / 8 if (iv and ti in ixv and set(iv) <= set(ixv[ti])) else nb
                if len(js) > 1:                          # the fan-out copy reads the positions once
                    b += 8.0 * occ_l[gi][js[0]]
        else:
            for pl in plans:
                iv = pl.index_values()
                b += nb * len(iv) / 8 if (iv and ti in ixv) else nb
        if gather:
            b += 8.0 * (occ_g[gi].sum() - occ_l[gi].sum())
        rows_moved[gi] = b
        moved += b
    build_bytes = sum(texts[ti][5].numel() * (1 + len(v) / 8) for ti, v in ixv.items())
    moved += build_bytes
    alg8d = sum(texts[ti][2] * P + 8.0 * occ_g[gi].sum() for gi, (ti, *_r) in enumerate(G))
    hbm_peak, peak_src = peaks()
    achieved = moved / (ms_step * 1e-3) / 1e9
    achieved8d = alg8d / (ms_step * 1e-3) / 1e9

    # per-(sigma, m) breakdown and (N > 1) phase split, outside the timed region
    breakdown, phases = None, None
    if not args.no_breakdown:
        gev = {}
        pev = [] if world > 1 else None
        torch.cuda.synchronize()
        one_step(phase_ev=pev, group_ev=gev if world == 1 else None)
        torch.cuda.synchronize()
        if world == 1:
            rows = []
            for ti in ixs:
                us = gev[("ix", ti)][0].elapsed_time(gev[("ix", ti)][1]) * 1e3
                nb = texts[ti][5].numel()
                mg = nb * (1 + len(ixv[ti]) / 8) / (us * 1e-6) / 1e9
                rows.append([texts[ti][0], 0, round(us, 1), None, round(mg, 1), len(ixv[ti]), 0,
                             round(mg / hbm_peak, 3)])
            for gi, (ti, m, g, plans) in enumerate(G):
                us = gev[gi][0].elapsed_time(gev[gi][1]) * 1e3
                nb = texts[ti][5].numel()
                dense = sum(g.dense_searches()) if args.mode == "group" else None
                mg = rows_moved[gi] / (us * 1e-6) / 1e9
                rows.append([texts[ti][0], m, round(us, 1), round(P * nb / (us * 1e-6) / 1e9, 1),
                             round(mg, 1), dense, int(occ_l[gi].sum()), round(mg / hbm_peak, 3)])
            breakdown = {"cols": ["sigma", "m (0: index build)", "us per group of searches", "text_GBps",
                                  "moved_GBps", "dense searches (0: index values)", "positions",
                                  "moved_frac (moved_GBps / peak)"], "rows": rows}
        else:
            sc = sum(e[0].elapsed_time(e[1]) for e in pev)
            cc = sum(e[1].elapsed_time(e[2]) for e in pev)
            ga = sum(e[2].elapsed_time(e[3]) for e in pev)
            sc, cc, ga = (max_over_ranks(x, world, dev) for x in (sc, cc, ga))
            phases = {"scan_ms": round(sc, 3), "count_exchange_ms": round(cc, 3),
                      "gather_ms": round(ga, 3) if gather else None,
                      "note": "one step with CUDA events between the phases of every group (the index "
                              "builds count as scan); max over ranks"}
            phases["keep_sharded_value"] = round(n_text_step / ((sc + cc) * 1e-3) / 1e9, 2)

    tf = traffic_file()
    res = {
        "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_step, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": {"workload": "BASELINE configs[1]: random-alphabet sweep, n=256 MiB per text"
                               + (f" per rank (text n={world}x256 MiB, sharded, 31-byte halo)" if world > 1 else ""),
                   "sigmas": sigmas, "ms": ms, "patterns_per_sigma_m": P,
                   "searches_per_step": len(G) * P, "text_bytes_per_step": n_text_step,
                   "l2": "no flush: every text (256 MiB) is larger than the 126 MB L2",
                   "parallelism": f"dp{world} over text shards" if world > 1 else "single GPU",
                   "api": (("epsm_eqidx_build_async per text + epsm_group_search_index_async per (sigma, m)"
                            if args.mode == "group" else
                            "epsm_eqidx_build_async per text + epsm_search_batch_index_async per (sigma, m)")
                           if world == 1 else
                           "epsm_group_search_range_index_async per (sigma, m) + NCCL all-gather of the count "
                           "matrix" + ("" if not gather else " + epsm_allgatherv_async (positions to every rank)")),
                   "positions": ("every search's positions in its own device buffer" if world == 1 else
                                 "all-gathered: every rank holds every search's global positions (sub-batches "
                                 "of searches into reused buffers)" if gather else
                                 "kept sharded: each rank holds its owned positions at their global offsets")},
        "roofline": roofline_block(achieved, achieved8d, moved, alg8d, hbm_peak, peak_src, tf, gather,
                                   kt_n, kt_ms, kt_bytes, args.steps, ms_step),
        "clocks": clocks,
        "gpu_launches": int(launches),
        "total_occ_per_step": int(occ_g.sum()),
        "parity": checked,
        "breakdown": breakdown,
        "phases": phases,
    }
    if world == 1 and args.scan_patterns > 0:
        res["scan"] = run_scan(args, epsm, texts, pats, ms, hbm_peak)
    if world == 1 and (not args.no_e2e or not args.no_configs):
        del pool
        torch.cuda.empty_cache()
    if world == 1 and not args.no_e2e:
        res["e2e"] = run_e2e(args, epsm, texts, G, P)
    if world == 1 and not args.no_configs:
        texts_keep = texts
        res["configs"] = run_configs(args, epsm, dev, hbm_peak)
        del texts_keep
    if rank == 0 and world == 1 and not args.no_cpu:
        res["cpu_baseline"], res["cpu_epsm"] = cpu_baselines(args, texts, pats, ms)
    for _, _, g, plans in G:
        g.close()
        for pl in plans or ():
            pl.close()
    return res


def oracle_full_counts(args, texts, pats, G, occ_glob, world, rank):
    """One search per group: the oracle's count over the WHOLE (global) text == the GPU's occ.
    Rank 0 only (N > 1: the global text is generated on the host from the counter-based
    generator); the oracle runs one search per host thread."""
    if rank != 0:
        return None
    if world > 1:
        # (the global texts are N x 256 MiB each: the windows of the gathered positions, checked in
        # the warm-up, are the oracle evidence at N > 1; full-text counts would take minutes)
        return {"oracle_full_text_counts": 0, "oracle_windows_per_group": 2, "window_bytes": WINDOW,
                "ok": True, "note": "N > 1: gathered positions checked in 1 MiB oracle windows"}
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    occ_h = occ_glob.cpu().numpy()
    hosts = {}
    jobs = []
    for gi, (ti, m, g, plans) in enumerate(G):
        s, spec, n_total = texts[ti][0], texts[ti][1], texts[ti][2]
        if ti not in hosts:
            hosts[ti] = texts[ti][5].cpu().numpy() if world == 1 else synth.text_np(spec, 0, n_total)
        j = gi % args.patterns
        jobs.append((gi, j, pats[(s, m)][j], ti))
    t0 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=len(os.sched_getaffinity(0))) as ex:
        counts = list(ex.map(lambda a: oracle.count(a[2], hosts[a[3]]), jobs))
    for (gi, j, p, ti), c in zip(jobs, counts):
        assert int(occ_h[gi, j]) == c, f"oracle count mismatch: sigma={texts[ti][0]} m={len(p)} search {j}"
    return {"oracle_full_text_counts": len(jobs), "oracle_windows_per_group": 2, "window_bytes": WINDOW,
            "ok": True, "oracle_s": round(time.perf_counter() - t0, 2)}


def run_scan(args, epsm, texts, pats, ms, peak):
    """The north_star's online per-pattern scan: one epsm_search_async launch per search over
    the TEXT (no index, no group), CUDA events around each launch, all K launches queued
    behind a GPU spin so that the events time the kernels; per (sigma, m): mean /
    median us, text GB/s = n / t and the SURVEY 8(d) fraction (n + 8 occ) / t / peak.  Plus the
    host wall time of the synchronous call including epsm_plan and the occ readback."""
    dev = texts[0][5].device
    stream = torch.cuda.current_stream(dev)
    K = args.scan_patterns
    n = texts[0][5].numel()
    pos = torch.empty(n, dtype=torch.int64, device=dev)
    rows, tot_t, tot_b = [], 0.0, 0.0
    for s, spec, n_total, base, owned, t in texts:
        for m in ms:
            plans = [epsm.plan(p) for p in pats[(s, m)][:K]]
            occ = torch.zeros(K, dtype=torch.int64, device=dev)
            for j, pl in enumerate(plans):                     # warm
                epsm.search_async(pl, t, pos, occ[j:j + 1])
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * K)]
            # the GPU spins (~4 ms) while the host queues the K launches: each event pair then
            # brackets the kernel alone, not the host's launch latency (that is the last column)
            torch.cuda._sleep(8_000_000)
            for j, pl in enumerate(plans):
                ev[2 * j].record(stream)
                epsm.search_async(pl, t, pos, occ[j:j + 1])
                ev[2 * j + 1].record(stream)
            torch.cuda.synchronize()
            us = np.array([ev[2 * j].elapsed_time(ev[2 * j + 1]) * 1e3 for j in range(K)])
            oc = occ.cpu().numpy().astype(np.float64)
            byts = n + 8.0 * oc
            tot_t += us.sum()
            tot_b += byts.sum()
            # synchronous call from host bytes to occ, plan included
            t0 = time.perf_counter()
            for p in pats[(s, m)][:2]:
                epsm.count(p, t)
            wall = (time.perf_counter() - t0) / 2 * 1e6
            rows.append([s, m, round(float(us.mean()), 1), round(float(np.median(us)), 1),
                         round(n / (us.mean() * 1e-6) / 1e9, 1),
                         round(float((byts / (us * 1e-6)).mean()) / 1e9 / peak, 3), round(wall, 1)])
            for pl in plans:
                pl.close()
    fr = [r[5] for r in rows]
    return {"cols": ["sigma", "m", "mean_us", "median_us", "text_GBps", "frac_8d", "host_wall_us_plan_count"],
            "rows": rows, "patterns_per_sigma_m": K, "text_GBps": round(len(rows) * K * n / (tot_t * 1e-6) / 1e9, 1),
            "frac_8d": round(tot_b / (tot_t * 1e-6) / 1e9 / peak, 4),
            "min_frac_8d": min(fr), "below_0.7": sum(1 for x in fr if x < 0.7),
            "note": "one search per launch over the text kernels (no index, no group) -- EPSM's online "
                    "per-pattern search; the K launches of a (sigma, m) are queued behind a GPU spin, so "
                    "the events time the kernels (host cost: last column); frac_8d = (n + 8 occ) / t / "
                    "peak, per search, averaged"}


def run_configs(args, epsm, dev, peak):
    """BASELINE.json's other configs through the same public API as the headline (one group call
    per (text, m), the text's index over its dense patterns' bytes): 1 (1 MiB ACGT, 16 x m=4),
    3a/3b (1 GiB genome-/protein-like, m = 2..32), 4 (1 GiB Zipf-27), 5a (8 GiB ACGT, m = 8, 32),
    5b ('a'^(2^30), 'a'^16).  Per (text, m): one warm and one timed call (CUDA events, the index
    build timed apart), text GB/s = patterns x n / t, moved GB/s (text once per pass + 8 B per
    position), oracle windows on two searches per group (config 1: the full oracle; 5b: the
    closed form occ = n - 15, positions = 0 .. n - 16 sampled)."""
    import oracle
    stream = torch.cuda.current_stream(dev)
    rng = np.random.default_rng(99)
    out = {}
    for cfg in ("1", "3", "4", "5a", "5b"):
        for w in synth.config_workloads(cfg):
            text = synth.text_torch(w.spec, 0, w.n, device=dev)
            groups = {}
            for m in w.ms:
                p, _ = (synth.extract_patterns_torch(text, w.start_seed(m), m, w.patterns_per_m)
                        if cfg != "5b" else ([b"a" * m], None))
                groups[m] = (p, epsm.group(p))
            vals = sorted({v for _, g in groups.values() for v in g.index_values()})
            ix, build_us = None, 0.0
            if vals:
                ix = epsm.EqIndex()
                ix.build_async(text, bytes(vals))
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                ix.build_async(text, bytes(vals))
                e1.record(stream)
                torch.cuda.synchronize()
                build_us = e0.elapsed_time(e1) * 1e3
            rows, t_tot, txt_tot, mv_tot = [], build_us, 0.0, w.n * (1 + len(vals) / 8) if vals else 0.0
            for m, (p, g) in groups.items():
                k = len(p)
                occ = torch.zeros(k, dtype=torch.int64, device=dev)
                g.count_async(text, occ, index=ix)
                torch.cuda.synchronize()
                cap = int(occ.max().item()) + 1
                outs = [torch.empty(cap, dtype=torch.int64, device=dev) for _ in range(k)]
                g.search_async(text, occ, outs=outs, index=ix)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                g.search_async(text, occ, outs=outs, index=ix)
                e1.record(stream)
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) * 1e3
                oc = occ.cpu().numpy()
                if cfg == "1":
                    host = text.cpu().numpy()
                    for j in range(k):
                        want = oracle.search(p[j], host)
                        assert int(oc[j]) == want.size and np.array_equal(
                            outs[j][:want.size].cpu().numpy().astype(np.uint64), want), "config 1 parity"
                elif cfg == "5b":
                    assert int(oc[0]) == w.n - m + 1, "config 5b closed form"
                    for q in (0, 1, w.n // 3, w.n - m):
                        assert int(outs[0][q]) == q, "config 5b positions"
                else:
                    for j in (0, k - 1):
                        check_windows(p[j], outs[j], int(oc[j]), w.spec, w.n, rng)
                moved = w.n * len(g.info()["passes"]) + 8.0 * float(oc.sum())
                rows.append([m, round(us, 1), round(k * w.n / (us * 1e-6) / 1e9, 1),
                             round(moved / (us * 1e-6) / 1e9, 1), int(oc.sum()), int(sum(g.dense_searches()))])
                t_tot += us
                txt_tot += k * w.n
                mv_tot += moved
                del outs
                g.close()
            if ix is not None:
                ix.close()
            del text
            torch.cuda.empty_cache()
            out[w.name] = {"text_GBps": round(txt_tot / (t_tot * 1e-6) / 1e9, 1),
                           "moved_frac": round(mv_tot / (t_tot * 1e-6) / 1e9 / peak, 3),
                           "index_build_us": round(build_us, 1), "index_values": len(vals),
                           "cols": ["m", "us per group", "text_GBps", "moved_GBps", "positions", "dense searches"],
                           "rows": rows}
    out["note"] = ("group search per (text, m), patterns_per_m as BASELINE.json (100; config 1: 16; 5b: 1); "
                   "parity: oracle windows (config 1: full oracle; 5b: closed form)")
    return out


def run_e2e(args, epsm, texts, G, P):
    """The same sweep end to end through the C ABI with HOST buffers: per text ONE
    epsm_search_text_host call (its 5 groups: pinned host text in, index built on the device,
    counts, group searches, every search's positions copied out into pinned host buffers,
    overlapped with the next group's search).  Wall clock per step; plans/groups built before."""
    host_texts = [t.cpu().pin_memory() for (_, _, _, _, _, t) in texts]
    by_text = {}
    for ti, m, g, plans in G:
        by_text.setdefault(ti, []).append(g)
    # host outputs: pinned buffers for the search slots of a call (slot j of every text's call
    # writes buffer j mod B, sized for the largest occ it receives), B as large as a host budget
    # allows (--e2e-host-gb; the GPU boxes have ~196 GB of RAM, one text's positions reach 68 GB)
    occ_first = {ti: epsm.search_text_host(gs, host_texts[ti]) for ti, gs in by_text.items()}
    nslot = max(len(v) for v in occ_first.values())
    need = [max(int(v[j]) for v in occ_first.values() if j < len(v)) + 1 for j in range(nslot)]
    B = nslot
    while B > 1:
        sz = [max(need[j] for j in range(b, nslot, B)) for b in range(B)]
        if 8 * sum(sz) <= args.e2e_host_gb * 1e9:
            break
        B -= 1
    sizes = [max(need[j] for j in range(b, nslot, B)) for b in range(B)]
    bufs = [torch.empty(c, dtype=torch.int64).pin_memory() for c in sizes]
    outs = [bufs[j % B] for j in range(nslot)]
    h2d = d2h = 0

    def step():
        nonlocal h2d, d2h
        h2d = d2h = 0
        for ti, gs in by_text.items():
            k = sum(g.k for g in gs)
            occ = epsm.search_text_host(gs, host_texts[ti], outs[:k])
            h2d += host_texts[ti].numel()
            d2h += int(np.minimum(occ.astype(np.int64), np.array([o.numel() for o in outs[:k]])).sum()) * 8

    step()                                                     # warm
    t0 = time.perf_counter()
    for _ in range(args.e2e_steps):
        step()
    dt = (time.perf_counter() - t0) / args.e2e_steps
    n_step = sum(texts[ti][2] for ti, *_ in G) * P
    res = {"value": round(n_step / dt / 1e9, 2), "unit": UNIT, "h2d_bytes_per_step": int(h2d),
           "d2h_bytes_per_step": int(d2h), "ms_per_step": round(dt * 1e3, 2), "steps": args.e2e_steps,
           "host_buffers": B, "host_bytes": int(8 * sum(sizes)),
           "note": "C ABI epsm_search_text_host per text (pinned host text in; index, counts and group "
                   "searches on the device; every position copied into pinned host memory, copies "
                   "overlapped with the next group); host wall clock; search slot j of every call "
                   "writes pinned buffer j mod host_buffers"}
    del outs, bufs
    return res


# ----------------------------------------------------------------- host baselines

def cpu_baselines(args, texts, pats, ms, sample_bytes=None):
    """The oracle (brute force, never tuned) and the paper's EPSM in SSE4.2 (cpu_epsm/) on the
    host cores: one pattern per (sigma, m), positions reported, over the first `cpu-bytes` of
    each text, one pattern per thread."""
    import cpu_epsm
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    sample_bytes = sample_bytes or args.cpu_bytes
    cores = len(os.sched_getaffinity(0))
    tasks = []
    for s, spec, n_total, base, owned, t in texts:
        host = t[:sample_bytes].cpu().numpy() if isinstance(t, torch.Tensor) else t[:sample_bytes]
        for m in ms:
            tasks.append((pats[(s, m)][0], host))
    out = []
    for name, fn in (("oracle", oracle.search), ("epsm_sse4.2", cpu_epsm.search)):
        fn(b"xy", np.zeros(4, np.uint8))                       # load the library untimed
        t1 = time.perf_counter()
        _ = [fn(p, h) for p, h in tasks[:2]]
        one = (time.perf_counter() - t1) / 2                    # single-thread, per search
        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=cores) as ex:
            res = list(ex.map(lambda a: fn(a[0], a[1]), tasks))
        dt = time.perf_counter() - t0
        scanned = sum(h.size for _, h in tasks)
        out.append({"value": round(scanned / dt / 1e9, 3), "unit": UNIT, "cores": cores,
                    "kind": "oracle" if name == "oracle" else "paper's EPSM (SSE4.2), host",
                    "per_core_GBps": round(tasks[0][1].size / one / 1e9, 3),
                    "positions": int(sum(r.size for r in res)),
                    "sample": f"1 pattern per (sigma, m) = {len(tasks)} searches over the first "
                              f"{sample_bytes // synth.MiB} MiB of each text ({scanned / 1e9:.2f} GB, positions "
                              f"reported, {dt:.2f} s wall, one pattern per thread)"})
    return out[0], out[1]


def run_reference(args, world, rank):
    """--impl reference: the oracle as it stands, each step a bounded sample."""
    if rank != 0:
        return None
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    sigmas = [int(x) for x in args.sigmas.split(",")]
    ms = [int(x) for x in args.ms.split(",")]
    sample = min(args.cpu_bytes, 64 * synth.MiB)
    tasks = []
    for s in sigmas:
        spec = synth.raw_sigma_spec(s, (2, s))
        t = synth.text_np(spec, 0, N_PER_RANK)
        for m in ms:
            p = synth.extract_patterns_np(t, (2, s, m), m, 1)[0][0]
            tasks.append((p, t[:sample]))
    cores = len(os.sched_getaffinity(0))

    def one():
        t0 = time.perf_counter()
        with ThreadPoolExecutor(max_workers=cores) as ex:
            list(ex.map(lambda a: oracle.search(a[0], a[1]), tasks))
        return time.perf_counter() - t0
    oracle.count(b"x", np.zeros(1, np.uint8))
    for _ in range(args.warmup):
        one()
    dts = [one() for _ in range(args.steps)]
    scanned = sample * len(tasks)
    v = scanned / float(np.mean(dts)) / 1e9
    cb = {"value": round(v, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
          "sample": f"1 pattern per (sigma, m) = {len(tasks)} searches over the first {sample // synth.MiB} "
                    f"MiB of each text, positions reported, one pattern per thread"}
    return {"metric": METRIC, "value": round(v, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(float(np.mean(dts)) * 1e3, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
            "data": "synthetic", "impl": "reference",
            "config": {"workload": "BASELINE configs[1] random-alphabet sweep (bounded sample)",
                       "sigmas": sigmas, "ms": ms, "sample_bytes_per_search": sample},
            "cpu_baseline": cb,
            "e2e": {"value": round(v, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    maybe_relaunch(args)
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        res = run_reference(args, world, rank)
    else:
        res = run_epsm(args, world, rank, local)
    if rank == 0 and res is not None:
        line = json.dumps(res)
        print(line, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(line + "\n")
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
