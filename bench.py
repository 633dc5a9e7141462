#!/usr/bin/env python
"""bench.py — correction GB/s of the EXaCTz hot path on B200 (BASELINE.json metric).

One *step* = one full correction (exactz_correct: validate, reference of f,
every detect/edit round until no violation remains) of config C2 — the
512^3 float32 Nyx-like field at relative eps 1e-3 (BASELINE.json configs[1]) —
with inputs resident in HBM.  value = 4 * V / (max-over-ranks step time),
decimal GB/s of field processed (the paper's OT).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2]
  python bench.py --impl reference ...   # the CPU oracle arm

N > 1 (torchrun, one rank per GPU): the z-slab path (exactz_correct_sharded)
corrects the same field split over the ranks (scaling "strong").
Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MEASURED_PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback
METRIC = "correction GB/s (field bytes/wall time)"
KERNELS = {"stencil": "k_stencil_key2 (dense CheckConstraints stencil, R1-R3)",
           "events": "k_events / k_events_cached (C3 label walks, R5/R6)",
           "edit": "k_count_edit", "stencil_sparse": "k_act_list + k_stencil_list",
           "saddle_order": "k_saddle_order_vals (C2, R4)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N > 1: strong = the z-slabs of one config field; weak = one "
                         "config-sized field per rank stacked along z (P:577-589)")
    ap.add_argument("--impl", default="exactz", choices=["exactz", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ocr", action="store_true", help="skip the SZ-like OCR report")
    ap.add_argument("--cpu-sample", type=int, default=64, help="edge of the oracle's crop")
    ap.add_argument("--no-reformulated", action="store_true",
                    help="skip the extra timing of the reformulated constraints (NEXT-1)")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def workload_name(cfg, f):
    from synth import fields as S
    c = S.CONFIGS[cfg]
    shape = "x".join(str(d) for d in reversed(tuple(f.shape)))
    return f"{cfg} {c['name']} {shape} float32, rel eps {c['rel']:g}, uniform noise"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def crop(f, g, n):
    """the centred n^3 (or n x n 2D) crop: a bounded sample of the same field"""
    if f.dim() == 3 and f.shape[0] > 1:
        z0, y0, x0 = [(d - min(n, d)) // 2 for d in f.shape]
        sl = (slice(z0, z0 + min(n, f.shape[0])), slice(y0, y0 + min(n, f.shape[1])),
              slice(x0, x0 + min(n, f.shape[2])))
    else:
        m = n * 8
        y0, x0 = [(d - min(m, d)) // 2 for d in f.shape[-2:]]
        sl = (slice(None), slice(y0, y0 + min(m, f.shape[-2])), slice(x0, x0 + min(m, f.shape[-1])))
    return f[sl].contiguous(), g[sl].contiguous()


def oracle_run(f, g, xi):
    """the CPU oracle, as it stands (single thread), timed with a monotonic clock"""
    from oracle import oracle as O
    O.build()
    fn, gn = f.cpu().numpy(), g.cpu().numpy()
    t0 = time.perf_counter()
    r = O.correct(fn, gn, xi, 5)
    dt = time.perf_counter() - t0
    return dt, r


class Clocks:
    """nvidia-smi clocks/throttle sampling during the timed region"""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None
        self.path = os.path.join("/tmp", f"exactz_clocks_{os.getpid()}.csv")

    def start(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.index), "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self):
        if self.p is None:
            return None
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except Exception:
            self.p.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        mp = json.load(open(MEASURED_PEAKS))
        return float(mp["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


def golden_run(G, V_full):
    """the cached single-thread oracle run of the whole config (same input
    SHA-256; tools/make_golden.py), quoted with its host and date"""
    if not G:
        return None
    return {"value": 4.0 * V_full / G["oracle_s"] / 1e9, "unit": "GB/s", "seconds": G["oracle_s"],
            "iterations": G["iters"], "threads": G.get("oracle_threads", 1),
            "host_cpu": G.get("host_cpu"), "host_nproc": G.get("host_nproc"), "date": G.get("date"),
            "source": f"tests/golden/fullsize_{G['config']}.json (tools/make_golden.py)"}


def run_reference(args):
    """--impl reference: the CPU oracle on the box's host cores."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    f, g, xi, shas, golden = make_inputs(args.config)
    n = max(16, args.cpu_sample * 3 // 4)
    fs, gs = crop(f, g, n)
    fs, gs = fs.cpu(), gs.cpu()
    times = []
    iters = None
    for k in range(args.warmup + args.steps):
        dt, r = oracle_run(fs, gs, xi)
        if k >= args.warmup:
            times.append(dt)
            iters = r.iters
    V = fs.numel()
    ms = 1e3 * sum(times) / len(times)
    val = 4 * V / (ms / 1e3) / 1e9
    sample = (f"centred {'x'.join(str(d) for d in reversed(tuple(fs.shape)))} crop of the "
              f"{args.config} field, xi of the full field; oracle iters {iters}")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": workload_name(args.config, f) + " (bounded CPU sample)",
                   "sha256_f": shas["f"], "sha256_ghat": shas["ghat"]},
        "cpu_baseline": {"value": val, "unit": "GB/s", "cores": 1, "kind": "oracle",
                         "sample": sample, "host_cores": host_cores(), "cpu": cpu_model(),
                         "full_run": golden_run(golden, V_full=f.numel())},
        "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def free_port() -> int:
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def self_launch(args):
    """--gpus N > 1 without torchrun: start N ranks (one per GPU) the way the
    driver does.  Under torchrun, WORLD_SIZE must equal --gpus."""
    ws_env = os.environ.get("WORLD_SIZE")
    if ws_env is None:
        if args.gpus > 1:
            cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                   f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
            return subprocess.call(cmd)
        return None
    if int(ws_env) != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={ws_env}")
    return None


def sha256(t) -> str:
    import hashlib
    return hashlib.sha256(t.contiguous().cpu().numpy().tobytes()).hexdigest()


def make_inputs(cfg):
    """The config's field and its simulated decompression, generated on the
    CPU (one torch thread: bytes set by the seed alone, identical on every
    host), with their SHA-256 and the cached full-size oracle run of the
    same bytes when tests/golden holds one."""
    from synth import fields as S
    f, g, xi = S.make(cfg)
    shas = {"f": sha256(f), "ghat": sha256(g)}
    golden = None
    path = os.path.join(ROOT, "tests", "golden", f"fullsize_{cfg}.json")
    if os.path.exists(path):
        G = json.load(open(path))
        if G.get("sha_f") == shas["f"] and G.get("sha_ghat") == shas["ghat"] and "oracle_s" in G:
            golden = G
    return f, g, xi, shas, golden


def main():
    args = parse()
    rc = self_launch(args)
    if rc is not None:
        return rc
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    from __graft_entry__ import _load_builder
    _build = _load_builder()
    if rank == 0:
        _build.build()
    if ws > 1:
        dist.barrier()
    import paper_2604_01397_b200 as E
    from synth import fields as S

    weak = args.scaling == "weak" and ws > 1
    if weak:
        # weak scaling: rank r holds its own config-sized field
        # (same recipe, seed offset r), the ranks' fields stacked along z form
        # one (nx, ny, ws * nz) field; one xi for all (the smallest rank's
        # rel * range, so that min f >= xi holds on every rank)
        f, g, xi_r = S.make(args.config, device=dev, seed_offset=rank)
        t = torch.tensor([xi_r], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MIN)
        xi = float(t.item())
        f, g, _ = S.make(args.config, device=dev, seed_offset=rank, xi=xi)
        shas, golden = {"f": None, "ghat": None}, None
        V = f.numel() * ws
    else:
        f, g, xi, shas, golden = make_inputs(args.config)
        f, g = f.to(dev), g.to(dev)
        V = f.numel()
    wname = workload_name(args.config, f)
    if weak:
        wname += f" per rank, x{ws} stacked along z (weak scaling)"
    stream = torch.cuda.current_stream()
    sharded = ws > 1
    if weak:
        from paper_2604_01397_b200 import dist as D
        comm = D.open_comm(local)
        dims = (f.shape[2], f.shape[1], f.shape[0] * ws)
        f_run, g_run = f, g
        out = torch.empty_like(g_run)

        def step(profile=False):
            return E.exactz_correct_sharded(comm, f_run, g_run, dims, xi, out=out,
                                            stats_cap=1024)
    elif sharded:
        # strong scaling: the z-slabs of ONE field over the ranks (NCCL inside)
        from paper_2604_01397_b200 import dist as D
        comm = D.open_comm(local)
        z0, zc = D.slab_of(f.shape[0], ws, rank)
        dims = (f.shape[2], f.shape[1], f.shape[0])
        f_run, g_run = f[z0:z0 + zc].contiguous(), g[z0:z0 + zc].contiguous()
        del f, g
        torch.cuda.empty_cache()
        out = torch.empty_like(g_run)

        def step(profile=False):
            return E.exactz_correct_sharded(comm, f_run, g_run, dims, xi, out=out,
                                            stats_cap=1024)  # per-pass rows (paper: <= 612 passes)
    else:
        f_run, g_run = f, g
        out = torch.empty_like(g)

        def step(profile=False):
            return E.exactz_correct(f, g, xi, out=out, flags=E.PROFILE if profile else 0,
                                    stats_cap=1024)  # per-pass rows (paper: <= 612 passes)

    for _ in range(args.warmup):
        r0 = step()
    torch.cuda.synchronize()

    # ---------------- timed region: K steps, device time, max over ranks
    clocks = Clocks(local)
    clocks.start()
    launches0 = E.kernel_launches()
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    results = [step() for _ in range(args.steps)]
    ev1.record(stream)
    torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    launches = E.kernel_launches() - launches0
    ck = clocks.stop()
    # per-kernel-class event timing (EXACTZ_PROFILE) in separate, untimed steps
    prof_steps = max(1, min(args.steps, 2))
    profiled = [step(profile=True) for _ in range(prof_steps)]
    torch.cuda.synchronize()
    ms_total = ev0.elapsed_time(ev1)
    t = torch.tensor([ms_total], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_step = float(t.item()) / args.steps
    value = 4.0 * V / (ms_step / 1e3) / 1e9  # the whole field (strong scaling for N > 1)

    r = results[-1]
    iters = r.iters
    # Kernel classes timed with CUDA events on their launch streams
    # (EXACTZ_PROFILE, separate untimed steps).  algorithmic bytes per
    # launch: dense stencil 8.25 B per vertex;
    # C3 events 8 B per saddle walked + 8 B per link vertex walked from.
    agg = {}
    for res in profiled:
        for k, (ms, n, b) in res.kernels.items():
            a = agg.setdefault(k, [0.0, 0, 0])
            a[0] += ms
            a[1] += n
            a[2] += b
    peak, peak_src = peaks()

    def roof(cls):
        ms, n, b = agg.get(cls, (0.0, 0, 0))
        if not n or not ms:
            return None
        ach = (b / n) / ((ms / n) / 1e3) / 1e9
        return {"bound": "hbm", "kernel": KERNELS.get(cls, cls), "achieved": ach, "peak": peak,
                "unit": "GB/s", "frac": ach / peak, "traffic": None, "peak_source": peak_src,
                "bytes_per_launch": b / n, "ms_per_launch": ms / n, "launches_per_step": n / prof_steps,
                "share_of_step": ms / (ms_step * prof_steps)}

    # the dense stencil: the per-iteration kernel of north_star's 40 % gate and
    # the dominant kernel on the main stream
    roofline = roof("stencil") or {"bound": "hbm", "achieved": None, "peak": peak, "unit": "GB/s",
                                   "frac": None, "traffic": None}
    roofline["classes"] = {k: {"ms": v[0] / prof_steps, "launches": v[1] / prof_steps,
                               "GB/s": (v[2] / (v[0] / 1e3) / 1e9) if v[0] else None}
                           for k, v in agg.items() if v[1]}
    roofline_events = roof("events")
    traffic_path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        tr = json.load(open(traffic_path))
        for key, rl in (("k_stencil", roofline), ("k_events", roofline_events)):
            ent = tr.get(key, {})
            if rl is None or not ent:
                continue
            rl["traffic"] = ent.get("bytes_per_launch")
            rl["traffic_source"] = tr.get("source")
            rl["ncu"] = {k: v for k, v in ent.items() if k != "bytes_per_launch"}
        # the dense stencil's issue rate: warp-instructions per launch (ncu,
        # profiles/traffic.json) over the live launch time, against 148 SMs x
        # 4 schedulers x 1 instr/clk at the measured SM clock
        wi = tr.get("k_stencil", {}).get("warp_instr_per_32_vertices")
        if wi and roofline.get("ms_per_launch"):
            try:
                mhz = float(json.load(open(MEASURED_PEAKS)).get("sm_max_mhz", 1965.0))
            except Exception:
                mhz = 1965.0
            instr = wi * V / 32.0
            ach = instr / (roofline["ms_per_launch"] / 1e3) / 1e9
            pk = 148 * 4 * mhz * 1e6 / 1e9
            roofline["issue"] = {"bound": "issue", "achieved": ach, "peak": pk,
                                 "unit": "G warp-instr/s", "frac": ach / pk,
                                 "warp_instr_per_launch": instr,
                                 "source": "instructions from ncu (traffic.json), time live"}
    except Exception:
        pass

    # ---------------- e2e: host buffers in, host result out, every step
    fh, gh = f_run.cpu().pin_memory(), g_run.cpu().pin_memory()
    oh = torch.empty_like(gh).pin_memory()

    def e2e_step():
        if sharded:  # H2D of this rank's slab, the sharded call, D2H of its result
            fd = fh.to(dev, non_blocking=True)
            gd = gh.to(dev, non_blocking=True)
            rr = E.exactz_correct_sharded(comm, fd, gd, dims, xi, out=out)
            oh.copy_(out, non_blocking=True)
            return rr
        return E.exactz_correct_host(fh, gh, xi, out=oh)  # copies inside the C call

    e2e_step()  # warm
    ke = max(1, min(args.steps, 3))
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(ke):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1) / ke], dtype=torch.float64, device=dev)
    if ws > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item())
    same = bool(torch.equal(oh.view(torch.int32), out.cpu().view(torch.int32)))

    # ---------------- the reformulated constraints, same workload
    reform = None
    if not args.no_reformulated:
        def rstep():
            if sharded:
                return E.exactz_correct_sharded(comm, f_run, g_run, dims, xi, out=out,
                                                flags=E.REFORMULATED)
            return E.exactz_correct(f_run, g_run, xi, out=out, flags=E.REFORMULATED)
        rstep()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        r0e, r1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        kr = max(1, min(args.steps, 3))
        r0e.record(stream)
        for _ in range(kr):
            rr = rstep()
        r1e.record(stream)
        torch.cuda.synchronize()
        tr = torch.tensor([r0e.elapsed_time(r1e) / kr], dtype=torch.float64, device=dev)
        if ws > 1:
            dist.all_reduce(tr, op=dist.ReduceOp.MAX)
        reform = {"value": 4.0 * V / (float(tr.item()) / 1e3) / 1e9, "unit": "GB/s",
                  "ms_per_step": float(tr.item()), "iterations": rr.iters,
                  "speedup_vs_original": ms_step / float(tr.item())}

    # ---------------- Theorem 1 at full size (NEXT-3; untimed): iterations <= N * D_max
    thm = None
    if not sharded:
        t0 = time.perf_counter()
        vb = E.exactz_vulnerability(f_run, g_run, xi)
        torch.cuda.synchronize()
        thm = {"D_max": vb["D_max"], "bound": 5 * vb["D_max"], "iterations": iters,
               "holds": iters <= 5 * vb["D_max"], "G_V_pct": 100.0 * vb["GV"] / V,
               "G_S_pct": 100.0 * vb["GS"] / V, "G_R_pct": 100.0 * vb["GR"] / V,
               "seed_edges": vb["seeds"], "sweeps": vb["sweeps"],
               "ms": 1e3 * (time.perf_counter() - t0)}

    # ---------------- the edit set E as a log (NEXT-4; untimed)
    elog = None
    if not sharded:
        ce = torch.empty(V, dtype=torch.uint8, device=dev)
        rr = E.exactz_correct(f_run, g_run, xi, out=out, edit_counts=ce)
        t0 = time.perf_counter()
        log0, ne = E.exactz_edit_log(g_run, rr.out, ce, xi, level=0)
        t1 = time.perf_counter()
        log3, _ = E.exactz_edit_log(g_run, rr.out, ce, xi, level=3)
        elog = {"entries": ne, "edit_pct": 100.0 * ne / V,
                "lossless_clamp_pct": 100.0 * float((ce == 6).sum()) / V,
                "bytes_raw": len(log0), "bytes_zstd3": len(log3),
                "bytes_per_entry_zstd3": len(log3) / max(ne, 1),
                "field_bytes_over_log_zstd3": 4.0 * V / len(log3),
                "encode_ms_raw": 1e3 * (t1 - t0)}
        del ce, log0, log3

    # ---------------- OCR against the SZ-like base stream (NEXT-4; untimed):
    # the same field decompressed through SZ-like bins (synth/szlike.py), its
    # base stream size, the correction of that input and its edit log
    ocr = None
    if not sharded and not args.no_ocr:
        from synth import szlike as Z
        del out
        torch.cuda.empty_cache()
        f_sz = f_run
        g_sz = S.decompress(f_sz, xi, 0, mode="sz")
        enc = Z.encode(f_sz, xi, g_sz)
        c_sz = torch.empty(V, dtype=torch.uint8, device=dev)
        r_sz = E.exactz_correct(f_sz, g_sz, xi, edit_counts=c_sz)
        lg, ne_sz = E.exactz_edit_log(g_sz, r_sz.out, c_sz, xi, level=3)
        ocr = {"input": "same f, ghat = SZ-like bins 2 xi round(f / 2 xi) (decompress mode sz)",
               "base": "Lorenzo residuals of the bin codes, zigzag bytes + escapes, zstd -3",
               "base_bytes": enc["bytes"], "CR": 4.0 * V / enc["bytes"],
               "iterations": r_sz.iters, "status": r_sz.status,
               "edit_entries": ne_sz, "edit_pct": 100.0 * ne_sz / V,
               "edit_log_bytes_zstd3": len(lg),
               "OCR": 4.0 * V / (enc["bytes"] + len(lg))}
        del g_sz, c_sz, r_sz, lg, enc

    # ---------------- CPU baseline: the oracle on a bounded crop (rank 0, N = 1)
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        fs, gs = crop(f_run, g_run, args.cpu_sample)
        dt, ro = oracle_run(fs.cpu(), gs.cpu(), xi)
        cpu = {"value": 4 * fs.numel() / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
               "sample": (f"centred {'x'.join(str(d) for d in reversed(tuple(fs.shape)))} crop "
                          f"of the same field, xi of the full field; {dt:.1f} s, "
                          f"{ro.iters} iters"),
               "host_cores": host_cores(), "cpu": cpu_model(),
               "full_run": golden_run(golden, V)}

    # ---------------- per-pass %HBM: algorithmic bytes of a pass
    # = 8.25 B per vertex the stencil evaluated (V in a dense pass, the active
    # set in a change-tracked one) + 14 B per edit + 8 B per saddle (R4) + 8 B
    # per C3 link vertex walked from; T_iter = the pass's GPU span (CUDA
    # events on the call's stream, exactz_iter_stats.ms).
    per_pass = None
    if not sharded and getattr(r, "pass_ms", None):
        pk_meas, _ = peaks()
        rows = [(t, e, row[1], lk) for t, e, row, lk in
                zip(r.pass_ms, r.pass_evaluated, r.stats, r.pass_links) if t > 0]
        balg = [8.25 * e + 14.0 * ap + 8.0 * r.n_saddles + 8.0 * lk for _, e, ap, lk in rows]
        ms_l = [t for t, *_ in rows]
        fr = [b / (t / 1e3) / 1e9 for b, t in zip(balg, ms_l)]
        tot = sum(balg) / (sum(ms_l) / 1e3) / 1e9
        dense = [x for x, (_, e, _, _) in zip(fr, rows) if e == V]
        per_pass = {"passes": len(ms_l), "ms_min": min(ms_l), "ms_median": statistics.median(ms_l),
                    "ms_max": max(ms_l), "n_saddles": r.n_saddles,
                    "alg_bytes": "8.25 x evaluated + 14 E_t + 8 |S| + 8 x C3 link vertices",
                    "evaluated": [e for _, e, _, _ in rows],
                    "GBps": fr,
                    "GBps_median_pass": statistics.median(fr), "GBps_full_run": tot,
                    "frac_of_measured_median_pass": statistics.median(fr) / pk_meas,
                    "frac_of_measured_dense_passes": (statistics.median(dense) / pk_meas) if dense else None,
                    "frac_of_measured_full_run": tot / pk_meas,
                    "frac_of_8TBs_full_run": tot / 8000.0,
                    "passes_at_40pct_of_measured": sum(1 for x in fr if x >= 0.4 * pk_meas),
                    "max_frac_of_measured": max(fr) / pk_meas}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "strong" if sharded and not weak else "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": wname, "V": V, "xi": xi,
                       "sha256_f": shas["f"], "sha256_ghat": shas["ghat"],
                       "inputs": "generated on the host CPU (one torch thread), copied to HBM",
                       "iterations": iters, "status": r.status,
                       "ms_setup": r.ms_setup, "ms_loop": r.ms_loop,
                       "l2": f"inputs {4 * V / 1e6:.0f} MB per field > 126 MB L2 (no flush)",
                       "parallelism": (f"z-slabs x{ws} (NCCL send/recv + all-gather + "
                                       "all-reduce)") if sharded else "single GPU",
                       "edit_pct": elog["edit_pct"] if elog else None,
                       "mix": "worst case: uniform noise at the full amplitude xi (paper NYX: "
                              "0.73 % of the vertices edited, P:397-402)"},
            "iterations": iters,
            "hbm_frac": roofline["frac"],
            "per_pass": per_pass,
            "roofline": roofline,
            "roofline_events": roofline_events,
            "cpu_baseline": cpu,
            "e2e": {"value": 4.0 * V / (e2e_ms / 1e3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": 8 * V, "d2h_bytes_per_step": 4 * V,
                    "path": "torch H2D + exactz_correct_sharded + D2H per rank" if sharded
                    else "exactz_correct_host (pinned host buffers, copies inside the C call)",
                    "ms_per_step": e2e_ms, "bit_equal_to_device_run": same},
            "gpu_launches": launches,
            "reformulated": reform,
            "theorem1": thm,
            "edit_log": elog,
            "ocr": ocr,
            "clocks": ck,
            "version": E.version(),
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        comm.close()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
