#!/usr/bin/env python
"""bench.py — Poseidon per-layer gradient synchronisation on B200: per-iteration sync time,
parameters synchronised per second, and roofline fractions (BASELINE.json metric).

A "step" is one full-model synchronisation through the WFBP scheduler: every
layer of the model is triggered in backward order L..1 and synchronised with the scheme Algorithm 1
picks for it (SFB for FC layers, PS for CONV/BN layers), exactly as during training. Inputs
(factors u, v for FC layers; dense gradients for the rest; fp32 weights) are synthetic, resident in
HBM, with the shapes of the named torchvision architecture and per-GPU batch K (data-parallel weak
scaling: K is fixed per GPU, so the work per rank grows with N only through the K*N gathered
samples).

Default workload: config c3 = VGG19-22K (229,052,817 params), K = 32 per GPU — the north_star
target (BASELINE.json configs[3]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]
    python -m torch.distributed.run --nproc-per-node N --master-addr 127.0.0.1 bench.py --gpus N

Rank 0 prints ONE JSON line. `--impl reference` times the fp64 CPU oracle (oracle/, the only
reference this tier has) on a bounded sample of the same workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import synth_inputs as si  # noqa: E402

METRIC = "grad_sync_params_per_s"
UNIT = "params/s"


def default_bucket_mb(P, model=None):
    """PS unit size of the timed plan (--bucket-mb default), as measured on VGG19-22K (round 2):
    P = 1: 16 MiB (local applies; 64 MiB +0.8%); P = 2: 64 MiB (each fused cross-GPU unit costs
    ~17 us of fixed latency and the PS chain is exposed: 0.338 vs 0.375 ms with 16 MiB); P >= 4:
    16 MiB (0.366 vs 0.412 ms with 64 MiB — the big unit, issued last, ends the step).
    A model whose PS (dense) parameters dominate — FC parameters under half the dense ones, the
    scheduler's two-lane rule — takes 32 MiB at P = 2: four units, so two PS lanes (Inception-V3
    0.208 -> 0.189 ms; VGG19 / VGG19-22K are slower with 32 MiB: 0.264 / 0.338 ms)."""
    if P == 2 and model is not None:
        fc = sum(l.M * l.N for l in model.layers if l.kind == "fc")
        dense = sum(l.params for l in model.layers if l.kind != "fc")
        if fc < 0.5 * dense:
            return 32.0
    return 64.0 if P == 2 else 16.0


DEFAULT_BUCKET_MB = default_bucket_mb(1)
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}
NVLINK_GBS_PER_DIR = 770.0   # measured peer copy per direction (B200_PROFILING.md); 900 nominal


def load_nvlink(P):
    """Achievable per-direction NVLink bandwidth for P GPUs, measured by scripts/nvlink_peaks.py
    (nccl-tests style AG / RS busbw and the fused PS unit, plus — at P = 2 — copy-engine peer copies;
    profiles/nvlink_peaks.json); else the guide's peer-copy figure."""
    p = os.path.join(ROOT, "profiles", "nvlink_peaks.json")
    if P > 1 and os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        key = f"P{P}"
        if key in d:
            return float(d[key]["per_dir_gbs"]), f"measured (profiles/nvlink_peaks.json {key}: max of NCCL AG/RS busbw, the fused PS unit and copy-engine copies)"
        near = sorted(d, key=lambda k: abs(int(k[1:]) - P))
        if near:
            return float(d[near[0]]["per_dir_gbs"]), f"measured at {near[0]} (profiles/nvlink_peaks.json; no {key} entry)"
    return NVLINK_GBS_PER_DIR, "B200_PROFILING.md peer-copy figure (770 GB/s per direction)"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    return dict(PEAKS_FALLBACK, source="fallback (B200_PROFILING.md)")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=int(os.environ.get("WORLD_SIZE", "1")))
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="c3", choices=["c1", "c2", "c3", "c4"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "tf32", "f32"])
    ap.add_argument("--sequential", action="store_true", help="WFBP off: sync after the whole step")
    ap.add_argument("--max-ctas", type=int, default=0)
    ap.add_argument("--bucket-mb", type=float, default=None,
                    help="PS unit = consecutive dense layers up to this many MiB of fp32 (the paper "
                         "moves PS traffic in 2 MB KV pairs); default default_bucket_mb(P): 64 at "
                         "P = 2, else 16; 0 = one unit per layer")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-tf32", action="store_true", help="skip the extra tf32-factor measurement")
    ap.add_argument("--no-trace", action="store_true",
                    help="time the apply kernels with CUDA events (graph nodes) instead of device-side tracing")
    ap.add_argument("--no-symm", action="store_true",
                    help="P > 1: keep PS buffers and SFB gather buffers out of symmetric (NVLS) memory, i.e. use the stock NCCL collectives")
    ap.add_argument("--static-tiles", action="store_true", help="static round-robin reconstruction tiles")
    ap.add_argument("--ps-after-sfb", action="store_true",
                    help="P > 1: PS units wait for the SFB reconstructions instead of overlapping them")
    ap.add_argument("--eager", action="store_true",
                    help="issue every step from the host (default: replay the step as a CUDA graph)")
    ap.add_argument("--layers", action="store_true", help="also print a per-layer table to stderr")
    a = ap.parse_args()
    if a.warmup < 3:
        ap.error("--warmup must be >= 3")
    if a.dtype == "f32" and os.environ.get("POS_F32_FFMA") == "1":
        a.no_trace = True    # exact-fp32 mode: SIMT reconstruction, not traced — CUDA-event timing
    return a


# ------------------------------------------------------------------------------ accounting --
def plan_units(model, bucket_elems):
    """Synchronisation units: every FC layer alone (SFB); consecutive dense layers grouped into
    buckets of >= bucket_elems parameters (the paper's fixed-size KV pairs), a layer
    larger than that alone. bucket_elems = 0: one unit per layer (the paper's one syncer per layer)."""
    units, cur = [], None
    for l, ly in enumerate(model.layers):
        if ly.kind == "fc":
            if cur:
                units.append(cur)
                cur = None
            units.append({"kind": "fc", "layers": [l], "n": ly.params})
            continue
        if cur is None:
            cur = {"kind": "dense", "layers": [], "sizes": [], "n": 0}
        cur["layers"].append(l)
        cur["sizes"].append(ly.n)
        cur["n"] += ly.n
        if cur["n"] >= bucket_elems:
            units.append(cur)
            cur = None
    if cur:
        units.append(cur)
    return units


def unit_accounting(model, units, K, P, dtype):
    """Algorithmic bytes / flops per unit; never the dense all-reduce avoided."""
    sf = 2 if dtype == "bf16" else 4
    rows = []
    for u in units:
        if u["kind"] == "fc":
            ly = model.layers[u["layers"][0]]
            M, N = ly.M, ly.N
            KP = K * P
            rows.append({
                "name": ly.name, "scheme": "SFB", "params": ly.params,
                "hbm_a4": 8 * M * N + sf * KP * (M + N),
                "flop_a4": 2 * M * N * KP,
                "hbm_other": K * (M + N) * (2 + sf) + 8 * M + sf * KP * M,   # pack + bias
                "nvl": (P - 1) * K * (M + N) * sf,
            })
        else:
            S = _shard_len(u["n"], P)
            names = [model.layers[l].name for l in u["layers"]]
            rows.append({"name": names[0] + (f"..(+{len(names) - 1})" if len(names) > 1 else ""),
                         "scheme": "PS", "params": u["n"],
                         "hbm_a4": 0, "flop_a4": 0, "hbm_other": 12 * S,
                         "nvl": 2 * (P - 1) * S * 4 if P > 1 else 0})
    return rows


def _shard_len(n, P):
    """Rank 0's shard length from the library's shard table (the largest shard)."""
    import paper_1706_03292_b200 as pos
    lo, hi = pos.pos_shard_range(n, P, 0)
    return hi - lo


def roofline_times(rows, peaks, P, nvl_gbs=NVLINK_GBS_PER_DIR):
    hbm = peaks["hbm_gbs"] * 1e9
    tc = peaks["bf16_tflops"] * 1e12
    nvl = nvl_gbs * 1e9
    t_nvl = sum(r["nvl"] for r in rows) / nvl if P > 1 else 0.0
    t_k = sum(max(r["flop_a4"] / tc, (r["hbm_a4"] + r["hbm_other"]) / hbm) for r in rows)
    t_seq = sum((r["nvl"] / nvl if P > 1 else 0.0) + max(r["flop_a4"] / tc, (r["hbm_a4"] + r["hbm_other"]) / hbm)
                for r in rows)
    return max(t_nvl, t_k), t_seq, t_nvl, t_k


# ------------------------------------------------------------------------ the timed step --
def device_fill(gen, dtype):
    """Timing-run values, generated on the device: u = 2^-5 N(0,1), v = ReLU(N(0,1)),
    W ~ U(+-1/sqrt(N)), dense W ~ U(+-0.05), dense grads 2^-5 N(0,1)."""
    import torch
    fdt = torch.bfloat16 if dtype == "bf16" else torch.float32

    def fill(kind, layer, t, role):
        n = t.numel()
        if role == "W" and kind == "fc":
            t.copy_((torch.rand(t.shape, device=t.device, generator=gen) * 2 - 1) / math.sqrt(t.shape[1]))
        elif role == "b":
            t.zero_()
        elif role == "u":
            t.copy_((torch.randn(t.shape, device=t.device, generator=gen) * 2 ** -5).to(fdt))
        elif role == "v":
            t.copy_(torch.relu(torch.randn(t.shape, device=t.device, generator=gen)).to(fdt))
        elif role == "W":
            t.copy_((torch.rand(n, device=t.device, generator=gen) * 2 - 1) * 0.05)
        else:   # dense gradient
            t.copy_(torch.randn(n, device=t.device, generator=gen) * 2 ** -5)
    return fill


def register_units(pos, ctx, sch, model, units, K, dtype, fill, symm=True):
    """Register every synchronisation unit of the plan with the scheduler (SFB FC layers; dense
    buckets in symmetric memory when P > 1, so the fused NVLS kernels run), allocate its buffers and
    fill them with fill(kind, layer, tensor, role). Returns per-layer buffer records."""
    import torch
    P = ctx.world
    dev = torch.device("cuda", torch.cuda.current_device())
    in_dt = pos.POS_IN_BF16 if dtype == "bf16" else pos.POS_IN_F32
    fdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    bufs = [None] * len(model.layers)
    for un in units:
        if un["kind"] == "fc":
            l = un["layers"][0]
            ly = model.layers[l]
            M, N = ly.M, ly.N
            W = torch.empty(M, N, device=dev)
            fill("fc", l, W, "W")
            b = None
            if ly.bias:
                b = torch.empty(M, device=dev)
                fill("fc", l, b, "b")
            u = torch.empty(K, M, device=dev, dtype=fdt)
            v = torch.empty(K, N, device=dev, dtype=fdt)
            fill("fc", l, u, "u")
            fill("fc", l, v, "v")
            s = sch.add_fc(l, M, N, K, W, b, None, dtype=dtype, in_dtype=in_dt)
            assert s == pos.POS_SCHEME_SFB, (ly, s)   # Alg. 1 at these configs
            bufs[l] = {"kind": "fc", "W": W, "b": b, "u": u, "v": v}
        else:
            n = un["n"]
            Pn = pos.pos_padded_size(n, P)
            sy = P > 1 and symm       # the fused NVLS PS kernel needs symmetric W and grad
            W = ctx.sym_empty(Pn) if sy else torch.zeros(Pn, device=dev)
            g = ctx.sym_empty(Pn) if sy else torch.zeros(Pn, device=dev)
            off = 0
            for l, nl in zip(un["layers"], un["sizes"]):
                fill("dense", l, W[off:off + nl], "W")
                fill("dense", l, g[off:off + nl], "g")
                off += nl
            g0 = g.clone()
            sch.add_dense_bucket(un["layers"][0], un["sizes"], W, g)
            off = 0
            for l, nl in zip(un["layers"], un["sizes"]):
                bufs[l] = {"kind": "dense", "W": W[off:off + nl], "g": g[off:off + nl],
                           "g0": g0[off:off + nl], "n": nl, "Wflat": W, "gflat": g}
                off += nl
    return bufs


def make_step(sch, bufs, alpha):
    """One full-model synchronisation (Algorithm 2): begin, every layer triggered in backward order
    b^L .. b^1, end on the caller's stream."""
    L = len(bufs)

    def step(stream):
        sch.begin(alpha)
        for l in range(L - 1, -1, -1):
            bb = bufs[l]
            if bb["kind"] == "fc":
                sch.factors_ready(l, bb["u"], bb["v"], stream)
            else:
                sch.grad_ready(l, stream)
        sch.end(stream)
    return step


def isolated_kernels(pos, model, units, K, P, dtype, peaks):
    """Each hot-path kernel ALONE: back-to-back launches through the C ABI, captured
    in a CUDA graph and timed with two CUDA events around its replay on the launching stream (median
    of 3 replays), inputs larger than L2 rotated between launches;
    algorithmic bytes (flops) per launch / average launch time, against the measured peak.
      A4  reconstruct-and-apply, the model's largest SFB layer at K*P rows: 8MN + s(M+N)KP bytes
      A7  PS shard apply over the model's largest dense unit's shard: 12 bytes per element
      A2  factor pack of the largest SFB layer: K(M+N)(in + out) bytes."""
    import torch
    dev = torch.device("cuda", torch.cuda.current_device())
    dt = {"bf16": pos.POS_DT_BF16, "tf32": pos.POS_DT_TF32, "f32": pos.POS_DT_F32}[dtype]
    eb = 2 if dtype == "bf16" else 4
    fdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    hbm = peaks["hbm_gbs"]
    out = {}

    def timed(fn, n_launch=20, rot=2):
        # the launches are captured into one CUDA graph: host-side marshalling (ctypes, TMA
        # descriptor encoding) stays out of the measurement, which matters for microsecond kernels
        for i in range(3):
            fn(i % rot)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        cs = torch.cuda.Stream()
        cs.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
            for i in range(n_launch):
                fn(i % rot)
        torch.cuda.current_stream().wait_stream(cs)
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / n_launch)
        return statistics.median(ts)

    fcs = [model.layers[u["layers"][0]] for u in units if u["kind"] == "fc"]
    if fcs:
        ly = max(fcs, key=lambda l: l.M * l.N)
        M, N, KP = ly.M, ly.N, K * P
        R = pos.pos_factor_row_elems(M, N)
        G = (torch.randn(pos.pos_factor_slot_rows(KP, dt), R, device=dev) * 0.03).to(fdt)
        Ws = [torch.randn(M, N, device=dev) for _ in range(2)]
        b = torch.zeros(M, device=dev)
        ms = timed(lambda i: pos.pos_reconstruct_apply(M, N, KP, dt, G, Ws[i], b, -1e-3))
        byts = 8 * M * N + eb * KP * (M + N)
        out["a4_reconstruct_apply"] = {
            "layer": f"{ly.name} {M}x{N}, K*P={KP}", "us": ms * 1e3, "achieved_gbs": byts / ms / 1e6,
            "frac_hbm": byts / ms / 1e6 / hbm, "tflops": 2 * M * N * KP / ms / 1e9,
            "frac_bf16_peak": 2 * M * N * KP / ms / 1e9 / peaks["bf16_tflops"]}
        u = torch.randn(K, M, device=dev).to(fdt)
        v = torch.randn(K, N, device=dev).to(fdt)
        slots = [torch.empty(pos.pos_factor_slot_rows(K, dt) * R, device=dev, dtype=fdt) for _ in range(2)]
        ms = timed(lambda i: pos.pos_pack_factors(u, v, slots[i], dt), n_launch=50)
        byts = K * (M + N) * (eb + eb)
        out["a2_pack"] = {"layer": f"{ly.name} K={K}", "us": ms * 1e3, "achieved_gbs": byts / ms / 1e6,
                          "frac_hbm": byts / ms / 1e6 / hbm,
                          "note": "a few MB per launch: latency-bound (launch + one wave), not bandwidth-bound"}
        del G, Ws, slots
    dens = [u for u in units if u["kind"] == "dense"]
    if dens:
        n = max(u["n"] for u in dens)
        lo, hi = pos.pos_shard_range(n, P, 0)
        cnt = max(hi - lo, 1)
        n_rot = max(2, int(math.ceil(3 * 126e6 / (8 * cnt))))    # rotate > 3x L2 of W + g
        gs = [torch.randn(cnt, device=dev) for _ in range(n_rot)]
        Wx = [torch.randn(cnt, device=dev) for _ in range(n_rot)]
        ms = timed(lambda i: pos.pos_ps_apply(gs[i], Wx[i], cnt, -1e-3), rot=n_rot)
        out["a7_ps_apply"] = {"elements": cnt, "us": ms * 1e3, "achieved_gbs": 12 * cnt / ms / 1e6,
                              "frac_hbm": 12 * cnt / ms / 1e6 / hbm,
                              "note": "shard of the largest dense unit; the fused NVLS kernel (P > 1) "
                                      "moves its reduce / broadcast over NVLink instead"}
    return out


def head_start(steps, stream):
    """Keep the GPU busy (a spin kernel, ~50 us per step to be enqueued) while the host enqueues the
    timed steps, so a host hiccup cannot leave the device idle inside the timed region: the region
    then measures device time only (its start event is recorded after the spin)."""
    import torch
    with torch.cuda.stream(stream):
        torch.cuda._sleep(int(max(1, steps) * 100_000))   # ~50 us per step at ~2 GHz


def capture_ring(fn, main, n=4):
    """CUDA graphs of one step each: replaying them round-robin keeps n timing-event slots of the
    scheduler live (slot = iteration mod 4), so per-kernel timings stay measurable."""
    import torch
    gs = []
    cs = torch.cuda.Stream()
    cs.wait_stream(main)
    for _ in range(n):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=cs, capture_error_mode="thread_local"):
            fn(torch.cuda.current_stream())
        gs.append(g)
    main.wait_stream(cs)
    return gs


# ------------------------------------------------------------------------------ clocks ------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.proc = None
        self.marks = {}

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            self.samples.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self, name):
        self.marks[name] = time.time()

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0, t1):
        sel = [s for (t, s) in self.samples if t0 <= t <= t1 and len(s) >= 9]
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"], "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(s[1]) for s in sel if num(s[1]) is not None]
        mx = [num(s[2]) for s in sel if num(s[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in sel for i in range(4) if s[5 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sel),
                "power_w_max": max((num(s[3]) or 0.0) for s in sel)}


# ------------------------------------------------------------------------------ our arm -----
def _log(msg):
    if os.environ.get("POS_BENCH_VERBOSE"):
        print(f"[bench r{os.environ.get('RANK', '0')} {time.strftime('%H:%M:%S')}] {msg}", file=sys.stderr, flush=True)


def run_ours(a):
    import faulthandler
    import numpy as np
    import torch
    import torch.distributed as dist

    if os.environ.get("POS_BENCH_VERBOSE"):
        faulthandler.dump_traceback_later(float(os.environ.get("POS_BENCH_WATCHDOG", "90")), exit=True)

    import paper_1706_03292_b200 as pos

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == a.gpus, f"--gpus {a.gpus} but WORLD_SIZE {world}"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        _log("process group up")
        ctx = pos.Context.from_torch_distributed()
        _log("poseidon context up")
    else:
        ctx = pos.Context.from_unique_id(bytes(128), 1, 0)
    if a.max_ctas:
        ctx.set_max_ctas(a.max_ctas)
    P = world
    model_name, K = si.CONFIGS[a.config]
    model = si.load_model(model_name)
    L = len(model.layers)
    alpha = -0.01 / P

    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 * 1 + rank)
    if a.bucket_mb is None:
        a.bucket_mb = default_bucket_mb(P, model)
    units = plan_units(model, int(a.bucket_mb * 2 ** 20 / 4))
    # The timed region replays UNTRACED step graphs. In-step kernel times come from a second ring
    # of the same step captured with device-side tracing (the kernels stamp %globaltimer; no timing
    # events in the captured step), replayed after the timed region; --layers adds per-stage events
    # and a timeline; --no-trace times the apply stages with CUDA events instead
    sch = pos.Scheduler(ctx, L, timing=(True if a.layers else ("apply" if a.no_trace else False)),
                        trace=False, sequential=a.sequential,
                        symm=not a.no_symm, ps_after_sfb=a.ps_after_sfb, static_tiles=a.static_tiles)
    bufs = register_units(pos, ctx, sch, model, units, K, a.dtype, device_fill(gen, a.dtype),
                          symm=not a.no_symm)
    main = torch.cuda.current_stream()
    step = make_step(sch, bufs, alpha)

    def barrier():
        if world > 1:
            dist.barrier(device_ids=[local])

    def refresh_grads():
        for bb in bufs:
            if bb["kind"] == "dense":
                bb["g"].copy_(bb["g0"])

    def check_async(where):
        # a cross-GPU wait that exceeded the watchdog (POS_TIMEOUT_MS) or an asynchronous CUDA
        # error: fail loudly instead of timing steps whose waits each run into the timeout
        rc = ctx.async_error()
        if rc < 0:
            raise pos.PoseidonError(rc, f"bench ({where}, rank {rank})")

    # ---- warmup (untimed, eager: NCCL connections, launch plans) ----
    _log(f"{len(units)} units registered; warmup")
    for _ in range(a.warmup):
        step(main)
        torch.cuda.synchronize()
        check_async("warmup")
    _log("warmup done")
    graphs = g_e2e = run_e2e = None
    if a.eager:
        run = lambda i: step(main)
    else:
        graphs = capture_ring(step, main)
        _log("captured")
        run = lambda i: graphs[i % len(graphs)].replay()
        for i in range(len(graphs)):
            run(i)
    torch.cuda.synchronize()
    check_async("graph warmup")
    _log("graph warmup done")
    refresh_grads()      # reduce-scatter sums in place; start the timed region from fresh gradients
    torch.cuda.synchronize()
    if a.layers or a.no_trace:
        sch.timing_reset()

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.3)
    barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
    t_wall0 = time.time()
    head_start(a.steps, main)
    evs[0].record(main)
    h0 = time.perf_counter()
    for i in range(a.steps):
        run(i)
        evs[i + 1].record(main)
    host_ms = (time.perf_counter() - h0) * 1e3 / a.steps   # host enqueue cost per step
    torch.cuda.synchronize()
    barrier()
    t_wall1 = time.time()
    ms = evs[0].elapsed_time(evs[-1]) / a.steps
    per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(a.steps)]
    _log(f"timed region done: {ms:.4f} ms/step")
    check_async("timed region")
    if world > 1:
        t = torch.tensor([ms] + per_step, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)          # max over ranks (per step)
        ms, per_step = float(t[0].item()), [float(x) for x in t[1:].tolist()]
    ps_sorted = sorted(per_step)
    step_stats = {"median_ms": statistics.median(per_step),
                  "p90_ms": ps_sorted[min(len(ps_sorted) - 1, int(math.ceil(0.9 * len(ps_sorted))) - 1)],
                  "min_ms": ps_sorted[0], "max_ms": ps_sorted[-1],
                  "note": "per-step device time (CUDA events between consecutive steps), max over ranks per step"}
    # span of the reconstructions within the step (they overlap: two streams) — before timing(),
    # which retires the events in eager mode
    has_fc, has_dense = any(u["kind"] == "fc" for u in units), any(u["kind"] == "dense" for u in units)
    traced_ms = None
    trace_timeline = None
    if a.no_trace:    # CUDA-event timing of the apply stages (events inside the captured step)
        a4_span_ms = sch.timing_span(pos.POS_SCHEME_SFB) if has_fc else None
        ps_span_ms = sch.timing_span(pos.POS_SCHEME_PS) if has_dense else None
        unit_apply_ms = [sch.timing(un["layers"][0])[2] for un in units]
    timeline = sch.timeline(len(units)) if a.layers else None
    unit_times = [sch.timing(un["layers"][0]) for un in units] if a.layers else None
    if not a.no_trace:   # the same step, traced, replayed as often as the timed region
        sch.set_trace(True)
        if a.eager:
            run_t = lambda i: step(main)
        else:
            graphs_t = capture_ring(step, main)
            run_t = lambda i: graphs_t[i % len(graphs_t)].replay()
        for i in range(4):
            run_t(i)
        refresh_grads()
        torch.cuda.synchronize()
        sch.trace_reset()
        barrier()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        head_start(a.steps, main)
        r0.record(main)
        for i in range(a.steps):
            run_t(i)
        r1.record(main)
        torch.cuda.synchronize()
        traced_ms = r0.elapsed_time(r1) / a.steps
        a4_span_ms = sch.trace_span(pos.POS_SCHEME_SFB)[0] / 1e3 if has_fc else None
        ps_span_ms = sch.trace_span(pos.POS_SCHEME_PS)[0] / 1e3 if has_dense else None
        unit_apply_ms = [sch.trace(un["layers"][0])[0] / 1e3 for un in units]
        # the last traced step's apply kernels as [first CTA start, last CTA end] (%globaltimer),
        # relative to the earliest: a timeline with no events on the streams (rank 0's)
        stamps = [sch.trace_last(un["layers"][0]) for un in units]
        t0 = min(st for st, _ in stamps)
        trace_timeline = [[model.layers[un["layers"][0]].name + ("" if len(un["layers"]) == 1 else f"..(+{len(un['layers']) - 1})"),
                           "SFB" if un["kind"] == "fc" else "PS", round((st - t0) / 1e3, 1), round((en - t0) / 1e3, 1)]
                          for un, (st, en) in zip(units, stamps)]
        if world > 1:
            t = torch.tensor([traced_ms, a4_span_ms or 0.0, ps_span_ms or 0.0] + unit_apply_ms, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            v = t.tolist()
            traced_ms = v[0]
            a4_span_ms = v[1] if has_fc else None
            ps_span_ms = v[2] if has_dense else None
            unit_apply_ms = v[3:]
        graphs_t = None
        sch.set_trace(False)
    # clock soak: if the timed region was too short for the 50 ms sampler, keep the same load
    # running (untimed) for ~1 s so the clock record describes this workload under load
    soak_t0 = soak_t1 = None
    if (t_wall1 - t_wall0) < 1.0:
        soak_t0 = time.time()
        n_soak = max(1, int(1.0 / max(ms / 1e3, 1e-5)))
        for i in range(n_soak):
            run(i)
        torch.cuda.synchronize()
        soak_t1 = time.time()
    # the eager (no graph) step, for reference: host-launch bound for many-layer models
    eager_ms = None
    if not a.eager:
        torch.cuda.synchronize()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        head_start(a.steps, main)
        g0.record(main)
        for _ in range(a.steps):
            step(main)
        g1.record(main)
        torch.cuda.synchronize()
        eager_ms = g0.elapsed_time(g1) / a.steps
        if world > 1:
            t = torch.tensor([eager_ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            eager_ms = float(t.item())

    # ---- e2e: the same step through the public API, inputs from pinned host memory ----
    e2e = None
    if not a.no_e2e:
        host_in, h2d, d2h = [], 0, 0
        for bb in bufs:
            if bb["kind"] == "fc":
                hu, hv = bb["u"].cpu().pin_memory(), bb["v"].cpu().pin_memory()
                host_in.append((hu, hv))
                h2d += hu.numel() * hu.element_size() + hv.numel() * hv.element_size()
            else:
                hg = bb["g0"][:bb["n"]].cpu().pin_memory()
                host_in.append((hg,))
                h2d += hg.numel() * 4
        res_dev = [bb["b"] for bb in bufs if bb["kind"] == "fc" and bb["b"] is not None]
        res_host = [r.cpu().pin_memory() for r in res_dev]
        d2h = sum(r.numel() * 4 for r in res_host)

        def e2e_step(stream):
            sch.begin(alpha)
            for l in range(L - 1, -1, -1):
                bb = bufs[l]
                if bb["kind"] == "fc":
                    bb["u"].copy_(host_in[l][0], non_blocking=True)
                    bb["v"].copy_(host_in[l][1], non_blocking=True)
                    sch.factors_ready(l, bb["u"], bb["v"], stream)
                else:
                    bb["g"][:bb["n"]].copy_(host_in[l][0], non_blocking=True)
                    sch.grad_ready(l, stream)
            sch.end(stream)
            for r, h in zip(res_dev, res_host):
                h.copy_(r, non_blocking=True)

        if a.eager:
            run_e2e = lambda i: e2e_step(main)
        else:
            g_e2e = capture_ring(e2e_step, main)
            run_e2e = lambda i: g_e2e[i % len(g_e2e)].replay()
        for i in range(4):
            run_e2e(i)
        torch.cuda.synchronize()
        barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        head_start(a.steps, main)
        f0.record(main)
        for i in range(a.steps):
            run_e2e(i)
        f1.record(main)
        torch.cuda.synchronize()
        ms_e2e = f0.elapsed_time(f1) / a.steps
        if world > 1:
            t = torch.tensor([ms_e2e], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms_e2e = float(t.item())
        e2e = {"value": P * model.total_params / (ms_e2e / 1e3), "unit": UNIT, "ms_per_step": ms_e2e,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "note": "per step: H2D of every layer's factors/gradients from pinned host memory, each layer "
                       "triggered after its upload (backward order), D2H of the FC biases (the "
                       "step's only host-visible result: W stays device-resident, as in training)"
                       + ("" if a.eager else "; step captured as a CUDA graph")}
    # ---- the same step with tf32 factors (4-byte floats, the paper's element width) ----
    tf32 = None
    if a.dtype == "bf16" and not a.no_tf32:
        sch2 = pos.Scheduler(ctx, L, trace=True, symm=not a.no_symm)
        bufs2 = []
        for l, bb in enumerate(bufs):
            if bb["kind"] == "fc":
                b2 = dict(bb, u=bb["u"].float(), v=bb["v"].float())
                ly = model.layers[l]
                sch2.add_fc(l, ly.M, ly.N, K, bb["W"], bb["b"], None, dtype="tf32", in_dtype=pos.POS_IN_F32)
                bufs2.append(b2)
            else:
                bufs2.append(bb)
        for un in units:
            if un["kind"] == "dense":
                bb = bufs[un["layers"][0]]
                sch2.add_dense_bucket(un["layers"][0], un["sizes"], bb["Wflat"], bb["gflat"])
        step2 = make_step(sch2, bufs2, alpha)
        for _ in range(3):
            step2(main)
        g2 = capture_ring(step2, main)
        for i in range(len(g2)):
            g2[i].replay()
        refresh_grads()
        torch.cuda.synchronize()
        sch2.trace_reset()
        barrier()
        q0, q1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        head_start(a.steps, main)
        q0.record(main)
        for i in range(a.steps):
            g2[i % len(g2)].replay()
        q1.record(main)
        torch.cuda.synchronize()
        ms2 = q0.elapsed_time(q1) / a.steps
        span2 = sch2.trace_span(pos.POS_SCHEME_SFB)[0] / 1e3
        if world > 1:
            t = torch.tensor([ms2, span2], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms2, span2 = (float(x) for x in t.tolist())
        rows2 = unit_accounting(model, units, K, P, "tf32")
        b2_a4 = sum(r["hbm_a4"] for r in rows2)
        tf32 = {"ms_per_step": ms2, "value": P * model.total_params / (ms2 / 1e3), "unit": UNIT,
                "a4_span_ms": span2, "a4_achieved_gbs": b2_a4 / (span2 / 1e3) / 1e9,
                "a4_frac_hbm": b2_a4 / (span2 / 1e3) / 1e9 / load_peaks()["hbm_gbs"],
                "note": "factors gathered as fp32 and contracted with tcgen05 kind::tf32 (fp32 accumulate)"}
        g2 = None
        torch.cuda.synchronize()
        sch2.close()
    kern_iso = isolated_kernels(pos, model, units, K, P, a.dtype, load_peaks())
    clocks.stop()
    if soak_t0 is not None:
        clk = clocks.summary(soak_t0, soak_t1)
        clk["window"] = "untimed soak of the same step right after the timed region (timed region < 1 s)"
    else:
        clk = clocks.summary(t_wall0, t_wall1)
        clk["window"] = "timed region"

    # ---- accounting & roofline ----
    peaks = load_peaks()
    rows = unit_accounting(model, units, K, P, a.dtype)
    nvl_gbs, nvl_src = load_nvlink(P)
    t_pipe, t_seq, t_nvl, t_kern = roofline_times(rows, peaks, P, nvl_gbs)
    a4_bytes = sum(r["hbm_a4"] for r in rows)
    a4_flop = sum(r["flop_a4"] for r in rows)
    # per-launch basis (the contract's "bytes per launch / average launch duration"): algorithmic
    # bytes of the step's reconstructions over the sum of their launch durations (first CTA start to
    # last CTA end of each launch); the span of all of them (they overlap on two streams) is kept
    # beside it
    n_a4 = sum(1 for r in rows if r["scheme"] == "SFB")
    a4_ms_sum = sum(unit_apply_ms[i] for i, r in enumerate(rows) if r["scheme"] == "SFB")
    a4_ms = a4_ms_sum if a4_ms_sum else (a4_span_ms or 0.0)
    ps_bytes = sum(r["hbm_other"] for r in rows if r["scheme"] == "PS")
    ps_ms = sum(unit_apply_ms[i] for i, r in enumerate(rows) if r["scheme"] == "PS")
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tj = json.load(f)
        key = f"{a.config}_P{P}_{a.dtype}"
        if key in tj:
            traffic = tj[key].get("a4_dram_bytes_per_step")
    achieved = a4_bytes / (a4_ms / 1e3) / 1e9 if a4_ms > 0 else None
    span_achieved = a4_bytes / (a4_span_ms / 1e3) / 1e9 if a4_span_ms else None
    roof = {"kernel": ("sfb_tc_kernel (A4 reconstruct-and-apply, fp32 as 3xTF32: 3 tf32 rows per pair"
                       if a.dtype == "f32" else "sfb_tc_kernel (A4 reconstruct-and-apply")
                      + ", all SFB layers of one step)",
            "bound": "hbm", "achieved": achieved, "peak": peaks["hbm_gbs"], "unit": "GB/s",
            "frac": achieved / peaks["hbm_gbs"] if achieved else None,
            # per launch like `achieved` (the step's launches averaged); the step total beside it
            "traffic": traffic / n_a4 if (traffic and n_a4) else None,
            "traffic_per_step": traffic,
            "algorithmic_bytes_per_launch": a4_bytes / n_a4 if n_a4 else None,
            "algorithmic_bytes_per_step": a4_bytes, "kernel_ms_per_step": a4_ms,
            "launches_per_step": n_a4, "avg_launch_ms": a4_ms / n_a4 if n_a4 else None,
            "kernel_ms_note": ("per-launch durations from CUDA events around each apply stage inside the "
                               "timed step graphs (--no-trace), averaged and summed over the step's "
                               "launches; achieved = algorithmic bytes of those launches / that sum")
                              if a.no_trace else
                              ("per-launch durations from the device-side trace (%globaltimer stamped by "
                               "the kernels: first CTA start to last CTA end; no events in the captured "
                               "step) of a replay of the same step right after the (untraced) timed "
                               "region, as many steps, averaged and summed over the step's launches; "
                               "achieved = algorithmic bytes of those launches / that sum"),
            "span_ms": a4_span_ms, "span_achieved": span_achieved,
            "span_frac": span_achieved / peaks["hbm_gbs"] if span_achieved else None,
            "span_note": "first reconstruction CTA start to last one's end in a step (consecutive layers' "
                         "reconstructions overlap on two streams; PS applies share HBM inside it)",
            "traced_ms_per_step": traced_ms,
            "per_layer_ms": {model.layers[un["layers"][0]].name: unit_apply_ms[i]
                             for i, un in enumerate(units) if un["kind"] == "fc"},
            "peak_source": peaks["source"],
            "tensor_tflops": a4_flop / (a4_ms / 1e3) / 1e12 if a4_ms > 0 else None,
            "tensor_frac_of_bf16_peak": (a4_flop / (a4_ms / 1e3) / 1e12) / peaks["bf16_tflops"] if a4_ms > 0 else None,
            "ps_units_in_step": {"algorithmic_bytes_per_step": ps_bytes, "sum_of_unit_ms": ps_ms,
                                 "span_ms": ps_span_ms,
                                 "note": "PS units run concurrently with the reconstructions and with "
                                         "each other: their summed durations are not a kernel time; "
                                         "see kernels_isolated.a7_ps_apply"},
            "kernels_isolated": kern_iso,
            "step": {"t_roofline_pipelined_ms": t_pipe * 1e3, "t_roofline_sequential_ms": t_seq * 1e3,
                     "t_nvlink_ms": t_nvl * 1e3, "t_kernels_ms": t_kern * 1e3,
                     "frac_pipelined": (t_pipe * 1e3) / ms, "nvlink_gbs_per_dir": nvl_gbs,
                     "nvlink_source": nvl_src}}
    symm_on = P > 1 and not a.no_symm
    flags_on = symm_on and os.environ.get("POS_GATHER_FLAGS", "1") != "0" and a.dtype != "f32"
    n_launch = 0
    for r, un in zip(rows, units):
        if r["scheme"] == "SFB":
            # P = 1: pack + reconstruct-and-apply (bias fused); P > 1 (NVLS): multicast pack +
            # reconstruct, plus the ready-flag wait kernel in flag mode; NCCL path: + all-gather
            n_launch += 2 + (1 if flags_on else 0)
        elif symm_on:
            n_launch += 1                   # fused NVLS reduce + apply + multicast kernel
        else:
            lo, hi = pos.pos_shard_range(un["n"], P, rank)
            ln = hi - lo
            n_launch += (1 if ln >= 4 else 0) + (1 if ln % 4 else 0)
    # NEXT-3: the B200 time model beside Algorithm 1 for every FC layer (report only; the
    # scheduler follows Alg. 1, the paper's rule)
    choice = []
    for ly in model.layers:
        if ly.kind != "fc":
            continue
        s_b, t_s, t_p = pos.pos_scheme_times_b200(ly.M, ly.N, K, P, 2 if a.dtype == "bf16" else 4,
                                                  peaks["hbm_gbs"] * 1e9, nvl_gbs * 1e9,
                                                  peaks["bf16_tflops"] * 1e12)
        choice.append({"layer": ly.name, "alg1": pos.SCHEME_NAMES[pos.pos_choose_scheme(ly.M, ly.N, K, P)],
                       "b200_model": pos.SCHEME_NAMES[s_b], "t_sfb_us": t_s * 1e6, "t_ps_us": t_p * 1e6,
                       "t_adam_us": 1e6 * pos.pos_scheme_time_adam_b200(
                           ly.M, ly.N, K, P, 2 if a.dtype == "bf16" else 4, peaks["hbm_gbs"] * 1e9, nvl_gbs * 1e9,
                           peaks["bf16_tflops"] * 1e12)})
    out = {
        "metric": METRIC, "value": P * model.total_params / (ms / 1e3), "unit": UNIT,
        "n_gpus": P, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": a.dtype, "data": "synthetic (random factors/gradients/weights of the named architecture's shapes)",
        "config": {"workload": f"{model_name} full-model gradient sync ({a.config}), K={K}/GPU, "
                               f"{'sequential (WFBP off)' if a.sequential else 'WFBP'}",
                   "model_params": model.total_params, "layers": L,
                   "fc_layers_sfb": sum(1 for r in rows if r["scheme"] == "SFB"),
                   "dense_layers_ps": sum(1 for ly in model.layers if ly.kind != "fc"),
                   "ps_units": sum(1 for r in rows if r["scheme"] == "PS"),
                   "ps_bucket_mb": a.bucket_mb,
                   "collectives": ("nccl" if (P == 1 or a.no_symm) else "fused NVLS kernels (symmetric memory)") if P > 1 else "none (P = 1)",
                   "per_gpu_batch": K, "global_batch": K * P, "parallelism": f"dp{P}",
                   "l2": "inputs larger than L2 (fp32 weights alone are "
                         f"{4 * model.total_params / 2**20:.0f} MiB vs 126 MB L2)",
                   "nccl": {k: v for k, v in os.environ.items() if k.startswith("NCCL_")}},
        "model_params_per_s": model.total_params / (ms / 1e3),
        "host_enqueue_ms_per_step": host_ms,
        "launch_mode": "eager" if a.eager else "cuda_graph (4-graph ring, one step each)",
        "eager_ms_per_step": eager_ms,
        "step_stats": step_stats,
        "roofline": roof,
        "tf32": tf32,
        "clocks": clk,
        "e2e": e2e,
        "scheme_choice": choice,
        "trace_timeline_us": trace_timeline,
        "gpu_launches": n_launch * a.steps,
        "gpu_launches_note": "libposeidon kernels per timed region (NCCL kernels and cudaMemsetAsync not counted)",
    }
    if a.layers and rank == 0:
        print("unit name scheme params | mean pack/comm/apply us | timeline of the last step (us from the "
              "first unit's start): start packed gathered apply0 apply1 done", file=sys.stderr)
        for l, (r, lt, tl) in enumerate(zip(rows, unit_times, timeline)):
            lt = (lt[0], lt[1], unit_apply_ms[l])
            print(f"{l:3d} {r['name']:>20s} {r['scheme']:>3s} params={r['params']:>11d} pack={lt[0]*1e3:8.1f} "
                  f"comm={lt[1]*1e3:8.1f} apply={lt[2]*1e3:8.1f} | " +
                  " ".join(f"{x * 1e3:8.1f}" if x >= 0 else "       -" for x in tl), file=sys.stderr)
        out["timeline_us"] = [[round(x * 1e3, 1) for x in tl] for tl in timeline]
    cpu = None
    if rank == 0 and P == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline_sample(a.config, P, a.dtype, min_seconds=10.0)
    out["cpu_baseline"] = cpu
    if rank == 0:
        print(json.dumps(out), file=_JSON_OUT, flush=True)
    # captured graphs hold NCCL resources of the communicator: free them before finalising it
    graphs = g_e2e = run = run_e2e = None
    import gc
    gc.collect()
    torch.cuda.synchronize()
    sch.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


# ----------------------------------------------------------------- oracle (CPU) baseline ----
def _oracle_sample(config, P, dtype):
    """A bounded sample of the workload for the fp64 oracle: the model's 4096x4096 FC layer (or its
    largest FC <= 2^24 params) via SFB plus its first 8 dense layers via PS, P workers."""
    import numpy as np
    model_name, K = si.CONFIGS[config]
    model = si.load_model(model_name)
    fcs = [l for l in model.layers if l.kind == "fc" and l.M * l.N <= (1 << 24)]
    fc = max(fcs, key=lambda l: l.M * l.N)
    dense = [l for l in model.layers if l.kind == "dense"][:8]
    dt = "bf16" if dtype == "bf16" else "f32"
    Us, Vs = zip(*(si.stat_factors(si.rng(7, 0, p), K, fc.M, fc.N, dt) for p in range(P)))
    W = si.stat_weights(si.rng(7, 1), fc.M, fc.N)
    b = np.zeros(fc.M, np.float32)
    dense_in = [(si.stat_weights(si.rng(7, 2 + i), 1, l.n)[0],
                 [si.stat_dense_grad(si.rng(8, i, p), l.n) for p in range(P)]) for i, l in enumerate(dense)]
    params = fc.params + sum(l.n for l in dense)
    desc = (f"{model_name}: {fc.name} ({fc.M}x{fc.N}, SFB, K*P={K * P}) + first {len(dense)} dense layers (PS); "
            f"{params} params of {model.total_params}; P={P} workers")
    return (fc, Us, Vs, W, b, dense_in), params, desc


def _oracle_step(sample, alpha):
    from oracle import sync   # bench.py's cpu_baseline / reference arm may execute the oracle
    fc, Us, Vs, W, b, dense_in = sample
    sync.sfb_update(W, b, Us, Vs, alpha)
    for Wd, gs in dense_in:
        sync.ps_update(Wd, gs, alpha)


def _cores():
    try:
        from threadpoolctl import threadpool_info
        th = [i.get("num_threads") for i in threadpool_info() if i.get("user_api") == "blas"]
        if th:
            return int(max(th))
    except Exception:
        pass
    return os.cpu_count()


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline_sample(config, P, dtype, min_seconds=10.0):
    sample, params, desc = _oracle_sample(config, P, dtype)
    _oracle_step(sample, -0.01 / P)      # warm
    t0 = time.perf_counter()
    n = 0
    while True:
        _oracle_step(sample, -0.01 / P)
        n += 1
        if time.perf_counter() - t0 >= min_seconds:
            break
    dt = (time.perf_counter() - t0) / n
    return {"value": P * params / dt, "unit": UNIT, "cores": _cores(), "kind": "oracle",
            "sample": desc + f"; {n} repetitions, {dt * 1e3:.1f} ms each", "os_cpu_count": os.cpu_count(),
            "cpu_model": _cpu_model()}


def run_reference(a):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    P = a.gpus
    sample, params, desc = _oracle_sample(a.config, P, a.dtype)
    for _ in range(a.warmup):
        _oracle_step(sample, -0.01 / P)
    t0 = time.perf_counter()
    for _ in range(a.steps):
        _oracle_step(sample, -0.01 / P)
    dt = (time.perf_counter() - t0) / a.steps
    value = P * params / dt
    model_name, K = si.CONFIGS[a.config]
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": P,
           "steps": a.steps, "warmup": a.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64",
           "data": "synthetic (same generators as the GPU arm)",
           "config": {"workload": f"{model_name} full-model gradient sync ({a.config}), K={K}/GPU — oracle on a "
                                  "bounded sample (see cpu_baseline.sample)", "per_gpu_batch": K,
                      "global_batch": K * P, "parallelism": f"dp{P} (computed on host, rank 0)"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": _cores(), "kind": "oracle", "sample": desc,
                            "cpu_model": _cpu_model()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), file=_JSON_OUT, flush=True)


_JSON_OUT = sys.stdout


def main():
    # The driver reads ONE JSON line from stdout: route everything else that writes to fd 1 (NCCL's
    # version banner, library prints) to stderr, and print the result line on the saved stdout.
    global _JSON_OUT
    sys.stdout.flush()
    _JSON_OUT = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
