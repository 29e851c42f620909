"""bench.py -- the LCP MVP hot path of arXiv 2604.10089 on B200.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                  [--config 4] [--gmres-tol 1e-8] [--no-c5]

A step is one LCP matrix-vector product w = D^T M D lambda (every
row of SURVEY 8(a): contacts, D scatter + P^T, RHS single-layer pass, GMRES on the
completed double-layer equation with K1/K2/K3 + device Arnoldi, rigid read-out,
D^T gather) at BASELINE.json config c4 (216 spheres, p = 16, N = 117 504 surface
points), lambda resident in HBM.  Timing: CUDA events around each step on the
launching stream, L2 flushed (256 MiB write) between steps outside the events;
W untimed warm-up steps; max over ranks.  The c5 line (one all-pairs S+D layer
apply with near and self parts, 259 200 points) gives pair-interactions/s.

N > 1 (torchrun): the MVP is sharded over the ranks (strong scaling):
rank r owns Np/N spheres' operator rows, K1 runs an equal share of the symmetric kernel's units,
and each operator application does one NCCL reduce-scatter and one all-gather on the library's
own communicator, enqueued on its stream.  --replicas: N independent MVPs instead (weak scaling,
no data-path collective).

--impl reference times the CPU oracle (oracle/, the only other place bench.py
executes it) on a bounded sample of the same workload; rank 0 only.
"""
import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # 37.2: SMs x FP64 FMA lanes/clk x 2 x max clock
METRIC = "ms per LCP MVP (c4: 216 spheres, p=16)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--gmres-tol", type=float, default=1e-8)   # paper's hi-fidelity eps_gmres (R9)
    ap.add_argument("--gmres-tol-lo", type=float, default=1e-6)  # low fidelity of a standalone LCP: <= 1e-6 (offline, R36); online runs 1e-8
    ap.add_argument("--gmres-restart", type=int, default=100)
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--recycle", type=int, default=1)   # GMRES recycling inside the LCP solve (NEXT-3)
    ap.add_argument("--solvers", default="bi,mono,bb")  # comma list of bi, mono, bb (BB-PGD)
    ap.add_argument("--no-fmm", action="store_true")    # skip the N >> 3e5 FMM context run (NEXT-4)
    ap.add_argument("--fmm-order", type=int, default=10)
    ap.add_argument("--no-refine", action="store_true")  # skip the FMM-refinement MVP / solve at the bench config
    ap.add_argument("--refine-order", type=int, default=6)  # FMM order of the refinement's Krylov steps
    ap.add_argument("--no-paper", action="store_true")  # skip the paper-setting context runs (p=8/4)
    ap.add_argument("--replicas", action="store_true")  # N > 1: independent replicas instead of the sharded MVP
    ap.add_argument("--shard-callback", action="store_true")  # N > 1: sharded via torch.distributed callbacks
    ap.add_argument("--shard-world1", action="store_true")    # N = 1: the sharded NCCL code path on a one-rank communicator
    ap.add_argument("--shard-asym", action="store_true")  # sharded K1 as the one-directional kernel (no reduce-scatter)
    ap.add_argument("--sub-forcing", type=float, default=0.0)   # Bi-PQN inexact subproblems (off = R22)
    ap.add_argument("--lo-dense", type=int, default=2)  # Bi-PQN: A^ formed once (1), matrix-free (0), auto (2; R38)
    ap.add_argument("--c5-steps", type=int, default=3)
    ap.add_argument("--cpu-sample-targets", type=int, default=0)
    return ap.parse_args()


# ---------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), "--query-gpu=" + self.Q,
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except (OSError, FileNotFoundError):
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, reasons, mx, pw = [], set(), None, []
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx = float(r[1])
                pw.append(float(r[2]))
            except ValueError:
                continue
            for k, name in enumerate(names):
                if r[3 + k].lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "power_w_max": max(pw) if pw else None}


# ---------------------------------------------------------------- distributed plumbing
def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        backend = "nccl" if args.impl == "ours" else "gloo"
        dist.init_process_group(backend=backend)
    return ws, rank, local


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(ws, v, device):
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------- oracle timing (cpu_baseline / reference)
def oracle_kg(c, tol=1e-8):
    """The ORACLE's own GMRES iteration count for one LCP MVP at tolerance tol (its residual
    history: the c4 certificate MVP, or the c1-c3 fixtures' dense-A runs), else the closest
    record.  Returns (k_g, source label)."""
    path = os.path.join(ROOT, "tests", "fixtures", "c%d.npz" % c)
    if os.path.exists(path):
        z = np.load(path, allow_pickle=True)
        if "oracle_gmres_hist" in z:
            h = np.asarray(z["oracle_gmres_hist"])
            if (h <= tol).any():
                return int(np.argmax(h <= tol)) + 1, "oracle GMRES history of the c%d certificate MVP at %g" % (c, tol)
        if "gmres_iters_mob" in z:
            return int(z["gmres_iters_mob"]), "oracle mobility solve of the c%d fixture at 1e-13 (no 1e-8 history)" % c
    return 100, "assumed (no oracle record)"


def oracle_mvp_sample(cfg, k_g, n_targets=0, n_inc_sample=2000, seed=7, sd=False):
    """The oracle (oracle/: plain-C OpenMP direct sum for the coarse part, numpy for the near,
    self and GMRES vector work, exactly the operations oracle.mobility.gmres / oracle.layer.Disc
    perform per operator pass) timed on a bounded sample of one LCP MVP:
      far   oracle far_sum for n_targets of the N targets x all sources (exclusion lists as in
            Disc.apply), scaled by N / n_targets;
      near  the refined-rule application einsum for n_inc_sample incidences, scaled by n_inc;
      self  the self-block einsum over all spheres;
      gmres one modified Gram-Schmidt step against k_g/2 basis vectors (the average);
    ms per MVP = (k_g + 1) x (far + near + self + gmres).  The near tensors and self rows are
    precomputed geometry (like bpqn_geometry_init) and not timed; their values do not change
    the arithmetic cost, so the self/near einsums run on arrays of the right shapes."""
    from oracle import native
    from oracle.grid import sphere_grid
    from oracle.layer import near_pairs
    from oracle.nearquad import incidences
    native.build()
    p, a = cfg["p"], cfg["radius"]
    grid = sphere_grid(p, a)
    nq = grid["xi"].shape[0]
    npn = cfg["np"]
    X = (cfg["centers"][:, None, :] + a * grid["xi"][None]).reshape(-1, 3)
    NRM = np.tile(grid["xi"], (npn, 1))
    W = np.tile(grid["w"], npn)
    N = X.shape[0]
    sphere_of = np.repeat(np.arange(npn), nq)
    dnear = 4.0 * np.pi * a / p
    inc = incidences(X, sphere_of, cfg["centers"], a, dnear, near_pairs(cfg["centers"], a, dnear))
    excl = [[] for _ in range(N)]
    for i, m in inc:
        excl[i].append(m)
    rng = np.random.default_rng(seed)
    q = rng.standard_normal((N, 3))
    f = rng.standard_normal((N, 3)) if sd else None   # S+D layer apply (c5): both densities
    n_targets = n_targets or max(1, N // 8)
    idx = np.sort(rng.choice(N, size=min(n_targets, N), replace=False))
    excl_ptr = np.zeros(idx.size + 1, dtype=np.int64)
    ex = []
    for k, t in enumerate(idx):
        ex.extend(excl[t])
        excl_ptr[k + 1] = len(ex)
    t0 = time.perf_counter()
    native.far_sum(X[idx], sphere_of[idx], excl_ptr, np.array(ex, dtype=np.int64), npn, nq, X, NRM, W, f, q,
                   cfg["mu"])
    t_far = (time.perf_counter() - t0) * N / idx.size
    nb = p * p + 2 * p
    ns = min(n_inc_sample, len(inc))
    t_near = 0.0
    if ns:
        T = rng.standard_normal((ns, 3, 3, nb))
        cf = rng.standard_normal((ns, nb, 3))
        out = np.zeros((ns, 3))
        t0 = time.perf_counter()
        np.add.at(out, np.arange(ns), np.einsum("kabn,knb->ka", T, cf))
        t_near = (time.perf_counter() - t0) * len(inc) / ns * (2 if sd else 1)
    D = rng.standard_normal((nq, 3, nq, 3))
    t0 = time.perf_counter()
    np.einsum("iajb,njb->nia", D, q.reshape(npn, nq, 3))
    t_self = (time.perf_counter() - t0) * (2 if sd else 1)
    kb = max(1, k_g // 2)
    t_gm = 0.0
    if k_g > 0:
        V = [rng.standard_normal(3 * N) for _ in range(kb)]
        w = rng.standard_normal(3 * N)
        t0 = time.perf_counter()
        for v in V:
            h = np.dot(v, w)
            w = w - h * v
        t_gm = time.perf_counter() - t0
    per_pass = t_far + t_near + t_self + t_gm
    passes = k_g + 1
    return dict(ms=per_pass * passes * 1e3, passes=passes, N=N, n_inc=len(inc), n_targets=int(idx.size),
                per_pass_s=dict(far=t_far, near=t_near, self=t_self, gmres=t_gm))


def cores_used():
    return int(os.environ.get("OMP_NUM_THREADS", os.cpu_count() or 1))


def cpu_desc():
    model = ""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return model


def run_reference(args, ws, rank):
    from synth import make_config
    if rank != 0:
        return
    cfg = make_config(args.config)
    k_g, src = oracle_kg(args.config, args.gmres_tol)
    times = []
    for _ in range(args.warmup):
        oracle_mvp_sample(cfg, k_g, args.cpu_sample_targets)
    for _ in range(args.steps):
        r = oracle_mvp_sample(cfg, k_g, args.cpu_sample_targets)
        times.append(r["ms"])
    v = float(np.mean(times))
    sample = ("oracle per-pass cost on a bounded sample (far: %d of %d targets x all sources, plain-C OpenMP; near: "
              "2000 of %d incidences; self: all spheres; GMRES MGS at k_g/2) x (k_g + 1 = %d) passes, k_g = the "
              "oracle's own iterations at tol %g (%s); host %s" %
              (r["n_targets"], r["N"], r["n_inc"], r["passes"], args.gmres_tol, src, cpu_desc()))
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "ms", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": v, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": "c%d LCP MVP" % args.config, "spheres": cfg["np"], "p": cfg["p"], "N": r["N"],
                       "gmres_tol": args.gmres_tol},
            "cpu_baseline": {"value": v, "unit": "ms", "cores": cores_used(), "kind": "oracle", "sample": sample,
                             "per_pass_s": r["per_pass_s"]},
            "e2e": {"value": v, "unit": "ms", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------- our arm
def run_ours(args, ws, rank, local):
    import torch
    import paper_2604_10089_b200 as bp
    from synth import make_config

    if not torch.cuda.is_available():
        raise SystemExit("bench.py: no CUDA device (the product has no CPU fallback)")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    stream = torch.cuda.current_stream(dev)
    cfg = make_config(args.config)
    t0 = time.time()
    g = bp.Geometry(cfg["centers"], cfg["p"], cfg["radius"], cfg["mu"])
    torch.cuda.synchronize()
    t_init = time.time() - t0
    pairs, nrm, gaps = bp.contacts(g, cfg["delta"])
    nc = g.nc
    shard = (ws > 1 and not args.replicas) or args.shard_world1
    if shard and ws == 1:   # self-test of the sharded path: one-rank NCCL communicator
        bp.geometry_shard_nccl(g, 0, 1, bp.nccl_unique_id(), symmetric=not args.shard_asym)
    elif shard:   # strong scaling of one MVP: each rank owns Np/N spheres' rows
        if args.shard_callback:
            bp.geometry_shard(g, rank, ws, symmetric=not args.shard_asym)
        else:
            import torch.distributed as dist
            uid = [bp.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(uid, src=0)
            bp.geometry_shard_nccl(g, rank, ws, uid[0], symmetric=not args.shard_asym)
    rng = np.random.default_rng(20260000 + args.config + 2000)     # synth.lambda_test recipe
    lam_h = rng.uniform(0.0, 1.0, size=nc)
    lam = torch.tensor(lam_h, dtype=torch.float64, device=dev)
    w = torch.empty(nc, dtype=torch.float64, device=dev)
    gm = bp.default_gmres_opts(tol=args.gmres_tol, restart=args.gmres_restart)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        bp.contacts(g, cfg["delta"])                  # A1 (K5) every step
        _, st = bp.lcp_mvp(g, lam, out=w, gmres=gm)   # A2-A5
        return st

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    bp.profile_reset(g, events=True)
    launches0 = bp.profile_get(g)["kernel_launches"]
    clk = ClockSampler(local)
    clk.start()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    gm_iters = []
    barrier(ws)
    torch.cuda.synchronize()
    for k in range(args.steps):
        flush.fill_(float(k))
        ev[k][0].record(stream)
        st = step()
        ev[k][1].record(stream)
        gm_iters.append(st.iters)
    torch.cuda.synchronize()
    barrier(ws)
    clocks = clk.stop()
    prof = bp.profile_get(g)
    ms_steps = [a.elapsed_time(b) for a, b in ev]
    total_ms = max_over_ranks(ws, float(np.sum(ms_steps)), dev)
    ms_per_step = total_ms / args.steps
    per_unit = 1 if shard else ws       # replicas: ws MVPs per step; sharded: one MVP per step
    launches = prof["kernel_launches"] - launches0
    k_g = float(np.mean(gm_iters))
    n_pairs_step = (k_g + 1.0) * g.N * g.N      # nominal N^2 per operator pass (RHS S-pass + k_g D-passes)

    w_ref = w.clone()   # the direct MVP at the bench tolerance (reference for the FMM refinement key)

    # e2e: the same MVP through the C ABI from pinned HOST lambda to a HOST w
    lam_pin = torch.tensor(lam_h, dtype=torch.float64).pin_memory()
    w_pin = torch.empty(nc, dtype=torch.float64).pin_memory()
    e2e_ms = []
    for k in range(max(2, min(args.steps, 3))):
        flush.fill_(float(k))
        torch.cuda.synchronize()
        t0 = time.perf_counter()                      # host clock around the whole user-visible call
        lam.copy_(lam_pin, non_blocking=True)
        bp.contacts(g, cfg["delta"])
        bp.lcp_mvp(g, lam, out=w, gmres=gm)           # returns after the device work (stats are host values)
        w_pin.copy_(w, non_blocking=True)
        torch.cuda.synchronize()
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
    e2e_v = max_over_ranks(ws, float(np.mean(e2e_ms)), dev) / per_unit

    # one MVP at the parity tolerance (1e-12, R9) for context
    _, st12 = bp.lcp_mvp(g, lam, out=w, gmres=bp.default_gmres_opts(tol=1e-12, restart=args.gmres_restart))

    k1_ms = prof["ms_allpairs"] / max(1, prof["allpairs_launches"])
    k1_tflops = prof["allpairs_gflop"] / max(prof["ms_allpairs"], 1e-9)  # GFLOP/ms = TFLOP/s
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "k1_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    line = {
        "metric": METRIC, "value": ms_per_step / per_unit, "unit": "ms", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": False,
        "scaling": "strong" if shard else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c%d LCP MVP" % args.config, "spheres": cfg["np"], "p": cfg["p"], "N": g.N,
                   "contacts": nc, "gmres_tol": args.gmres_tol, "gmres_restart": gm.restart,
                   "gmres_iters_per_mvp": k_g, "near_incidences": g.n_incidences,
                   "l2": "flushed between steps (256 MiB write outside the per-step events)",
                   "parallelism": (("shard-targets (one-directional K1, all-gather per operator application)"
                                    if args.shard_asym else
                                    "shard (symmetric K1 units split, reduce-scatter + all-gather per operator "
                                    "application)") + (" via torch.distributed callbacks" if args.shard_callback
                                                       else " on the library's NCCL communicator") if shard
                                   else ("replicas" if ws > 1 else "single GPU")),
                   "geometry_init_s": round(t_init, 3)},
        "pair_interactions_per_s": n_pairs_step * (1 if shard else ws) / (ms_per_step * 1e-3),
        "ms_per_mvp_tol_1e-12": st12.ms, "gmres_iters_tol_1e-12": st12.iters,
        "kernel_split_ms_per_step": {"k1_allpairs": prof["ms_allpairs"] / args.steps,
                                     "k2_near": prof["ms_near"] / args.steps,
                                     "k3_self": prof["ms_self"] / args.steps},
        "roofline": {"kernel": "k1_allpairs", "bound": "alu", "achieved": k1_tflops, "peak": FP64_PEAK_TFLOPS,
                     "unit": "TFLOP/s", "frac": k1_tflops / FP64_PEAK_TFLOPS, "traffic": traffic,
                     "k1_ms_per_launch": k1_ms,
                     "peak_source": "derived FP64 DFMA peak 148 SM x 64 lanes x 2 x 1.965 GHz (DESIGN.md); "
                                    "measured DFMA microbenchmark 37.0 (baseline/measured_fp64.json)"},
        "clocks": clocks,
        "gpu_launches": int(launches),
        "e2e": {"value": e2e_v, "unit": "ms", "h2d_bytes_per_step": 8 * nc, "d2h_bytes_per_step": 8 * nc},
    }
    if not args.no_solve:
        for k, meth in enumerate(args.solvers.split(",")):
            key = "lcp_solve" if k == 0 else "lcp_solve_" + meth
            line[key] = run_solve(args, cfg, g, pairs, nrm, gaps, dev, meth)
    del g
    torch.cuda.empty_cache()
    if not args.no_refine and not shard:
        line["mvp_fmm_refine"] = run_fmm_refine(args, cfg, dev, stream, lam, w_ref, ms_per_step / per_unit,
                                                pairs, nrm, gaps, flush)

    if not args.no_c5 and ws == 1:
        line["layer_apply_c5"] = run_c5(args, dev, stream)
    if not args.no_fmm and ws == 1:
        line["fmm_large"] = run_fmm_large(args, dev, stream)
    if not args.no_paper and ws == 1:
        line["paper_setting_6x6x6"] = run_paper_setting(args, dev, stream)

    if rank == 0 and ws == 1:
        k_g_or, src = oracle_kg(args.config, args.gmres_tol)
        r = oracle_mvp_sample(cfg, k_g_or, args.cpu_sample_targets)
        line["cpu_baseline"] = {
            "value": r["ms"], "unit": "ms", "cores": cores_used(), "kind": "oracle",
            "sample": "oracle per-pass cost on a bounded sample (far: %d of %d targets, plain-C OpenMP; near: 2000 of "
                      "%d incidences; self: all spheres; GMRES MGS at k_g/2) x (k_g + 1 = %d) passes, k_g = the "
                      "oracle's own iterations at tol %g (%s); host %s"
                      % (r["n_targets"], r["N"], r["n_inc"], r["passes"], args.gmres_tol, src, cpu_desc()),
            "per_pass_s": r["per_pass_s"]}
    if rank == 0:
        print(json.dumps(line), flush=True)


def run_solve(args, cfg, g, pairs, nrm, gaps, dev, meth="bi", relax=False):
    """One full LCP solve at the bench config: b from the Janus-slip non-collisional
    mobility solve, then Bi-PQN (Alg. 3) with the low fidelity at p_lo
    (or Mono-PQN when the config has none), paper-mode tolerances."""
    import torch
    import paper_2604_10089_b200 as bp
    gmo = bp.default_gmres_opts(tol=args.gmres_tol, restart=args.gmres_restart, recycle=int(args.recycle),
                                relax_fmm=int(relax))
    t0 = time.time()
    lo = None
    if meth == "bi" and cfg.get("p_lo"):
        lo = bp.Geometry(cfg["centers"], cfg["p_lo"], cfg["radius"], cfg["mu"])
        bp.set_contacts(lo, pairs, nrm, gaps)
    torch.cuda.synchronize()
    t_lo_init = time.time() - t0
    slip = bp.janus_slip(g, cfg["axes"], cfg["slip_B"])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b, st_b = bp.lcp_b(g, torch.tensor(cfg["F_nc"], device=dev), slip=slip, gmres=gmo)
    e1.record()
    torch.cuda.synchronize()
    ms_b = e0.elapsed_time(e1)
    o = bp.default_solve_opts(method=1 if lo is not None else (2 if meth == "bb" else 0), eps_kkt_abs=1e-8,
                              eps_kkt_rel=1e-8, k_max=500, sub_forcing=args.sub_forcing,
                              lo_dense=int(args.lo_dense) if meth == "bi" else 0)
    o.gm_hi = gmo
    o.gm_lo = bp.default_gmres_opts(tol=args.gmres_tol_lo, restart=args.gmres_restart, recycle=int(args.recycle))
    lam = torch.zeros(g.nc, dtype=torch.float64, device=dev)
    t0 = time.perf_counter()
    lam, rep, rc = bp.solve_lcp(g, lo, b, lam, opts=o)
    torch.cuda.synchronize()
    ms_solve = (time.perf_counter() - t0) * 1e3
    r = rep.as_dict()
    out = {"method": {"bi": "Bi-PQN", "mono": "Mono-PQN", "bb": "BB-PGD"}[meth] if (lo is not None or meth != "bi")
           else "Mono-PQN", "p_hi": cfg["p"], "p_lo": cfg.get("p_lo") if lo is not None else None,
           "gmres_recycling": bool(args.recycle), "gmres_tol_hi": args.gmres_tol,
           "gmres_tol_lo": args.gmres_tol_lo if lo is not None else None,
           "ms_b": ms_b, "gmres_iters_b": st_b.iters, "ms_solve": ms_solve, "ms_total": ms_b + ms_solve,
           "rc": rc, "lo_geometry_init_s": round(t_lo_init, 3),
           "negative_b_fraction": float((b < 0).double().mean().item()),
           "active_contacts": int((lam > 0).sum().item())}
    if relax:
        out["hi_mvps_with"] = "FMM refinement (relax_fmm = 1, fmm_order %d): Krylov steps with the FMM far field, " \
                              "every cycle from the direct residual" % args.refine_order
    out.update({k: r[k] for k in ("iterations", "hi_mvps", "lo_mvps", "lo_mvps_init", "lo_dense_columns",
                                  "lo_dense_gmres_iters", "ms_lo_dense", "e_mvps", "cost_ratio", "kkt_abs",
                                  "gmres_iters_hi", "gmres_iters_lo", "ms_hi", "ms_lo", "termination")})
    if lo is not None:
        lo.close()
    return out


def run_paper_setting(args, dev, stream):
    """Context only: the paper's online discretisation (hi p = 8, lo p = 4, eps_gmres 1e-8,
    P:531) on the 216-sphere c4 lattice (the paper's 6x6x6 runs): ms per LCP MVP,
    one LCP solve per method, and five full DVI time steps.  The paper reports
    collision resolution for 6x6x6 at 5d 0h 25m over 200 steps with BB-PGD (36.1 min per
    step) and 2.47x / 1.32x faster with Bi-PQN / Mono-PQN on 24 AMD Milan cores."""
    import torch
    import paper_2604_10089_b200 as bp
    from synth import make_config
    cfg = make_config(4)
    gm = bp.default_gmres_opts(tol=1e-8, restart=args.gmres_restart)
    hi = bp.Geometry(cfg["centers"], 8, cfg["radius"], cfg["mu"])
    lo = bp.Geometry(cfg["centers"], 4, cfg["radius"], cfg["mu"])
    pairs, nrm, gaps = bp.contacts(hi, cfg["delta"])
    bp.set_contacts(lo, pairs, nrm, gaps)
    lam = torch.tensor(np.random.default_rng(20262004).uniform(0, 1, hi.nc), device=dev)
    for _ in range(2):
        bp.lcp_mvp(hi, lam, gmres=gm)
    torch.cuda.synchronize()
    ms, its = [], []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, st = bp.lcp_mvp(hi, lam, gmres=gm)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        its.append(st.iters)
    gmo = bp.default_gmres_opts(tol=1e-8, restart=args.gmres_restart, recycle=1)
    slip = bp.janus_slip(hi, cfg["axes"], cfg["slip_B"])
    b, _ = bp.lcp_b(hi, torch.tensor(cfg["F_nc"], device=dev), slip=slip, gmres=gmo)
    solves = {}
    for meth, code in (("Bi-PQN", 1), ("Mono-PQN", 0), ("BB-PGD", 2)):
        o = bp.default_solve_opts(method=code, eps_kkt_abs=1e-8, eps_kkt_rel=1e-8, k_max=500,
                                  lo_dense=int(args.lo_dense) if code == 1 else 0)
        o.gm_hi = gmo
        o.gm_lo = gmo
        t0 = time.perf_counter()
        _, rep, rc = bp.solve_lcp(hi, lo if code == 1 else None, b, torch.zeros(hi.nc, dtype=torch.float64,
                                                                                  device=dev), opts=o)
        torch.cuda.synchronize()
        solves[meth] = {"ms": (time.perf_counter() - t0) * 1e3, "rc": rc, "iterations": rep.iterations,
                        "hi_mvps": rep.hi_mvps, "lo_mvps": rep.lo_mvps, "e_mvps": rep.e_mvps,
                        "kkt_abs": rep.kkt_abs, "ms_lo_dense": rep.ms_lo_dense}
    # one full DVI step (contacts, U_nc with slip, b, Bi-PQN, M D lambda, Euler, geometry update)
    C = np.ascontiguousarray(cfg["centers"].copy())
    A = np.ascontiguousarray(cfg["axes"].copy())
    # online steps: warm LCPs with few approaching contacts need few low-fidelity MVPs; the auto
    # mode (R38) keeps those matrix-free (forming A^ costs ~Nc lo solves)
    o = bp.default_solve_opts(method=1, eps_kkt_abs=1e-8, eps_kkt_rel=1e-8, k_max=500, lo_dense=int(args.lo_dense))
    o.gm_hi = gmo
    o.gm_lo = gmo
    steps = []
    for _ in range(5):   # five DVI steps of the 216-sphere suspension (NEXT-2)
        _, srep, src = bp.dvi_step(hi, lo, C, A, cfg["F_nc"], slip_B=cfg["slip_B"], dt=1e-2,
                                   delta=cfg["delta"], opts=o)
        steps.append({"rc": src, "ms": round(srep.ms_total, 1), "n_contacts": srep.n_contacts,
                      "active_contacts": srep.active_contacts, "hi_mvps": srep.lcp.hi_mvps,
                      "lo_mvps": srep.lcp.lo_mvps, "min_gap_after": srep.min_gap_after})
    out = {"workload": "c4 centres (6x6x6 lattice, 216 spheres) at the paper's online discretisation: "
                       "p=8 (N=%d), low fidelity p=4, eps_gmres 1e-8" % hi.N,
           "ms_per_mvp": float(np.mean(ms)), "gmres_iters_per_mvp": float(np.mean(its)), "lcp_solves": solves,
           "dvi_steps": {"dt": 1e-2, "ms_mean": float(np.mean([x["ms"] for x in steps])), "steps": steps},
           "paper_context": {"bb_pgd_collision_min_per_step": 7225.0 / 200.0,
                             "bi_pqn_collision_min_per_step": 7225.0 / 200.0 / 2.47,
                             "hardware": "24 cores AMD Milan, serial Matlab BIM + OpenMP STKFMM (P:528)",
                             "source": "PAPER.md Table 3 (P:613-629): 6x6x6 BB-PGD collision 5d 0h 25m / 200 steps"}}
    hi.close()
    lo.close()
    return out


def run_fmm_refine(args, cfg, dev, stream, lam, w_ref, ms_direct, pairs, nrm, gaps, flush):
    """The same c4 LCP MVP (same lambda, contacts, GMRES tolerance) with FMM-accelerated refinement
    (bpqn_gmres_opts.relax_fmm, NEXT-4; the paper's far field is an FMM): every Krylov step applies the
    operator with an order-`refine_order` FMM far field, each cycle starts from -- and the solve stops only on --
    the DIRECT residual b - A x (all-pairs K1), so the MVP meets the GMRES tolerance for the direct operator.
    Timed like the main MVP (CUDA events per MVP, L2 flushed between MVPs, contacts recomputed); its difference
    from the direct MVP is at the tolerance level.  Then the Bi-PQN solve with these hi MVPs."""
    import torch
    import paper_2604_10089_b200 as bp
    op = bp.default_disc_opts()
    op.fmm_order = args.refine_order
    t0 = time.time()
    g = bp.Geometry(cfg["centers"], cfg["p"], cfg["radius"], cfg["mu"], opts=op)
    torch.cuda.synchronize()
    t_init = time.time() - t0
    bp.contacts(g, cfg["delta"])
    w = torch.empty_like(w_ref)
    gm = bp.default_gmres_opts(tol=args.gmres_tol, restart=args.gmres_restart, relax_fmm=1)
    for _ in range(max(1, args.warmup)):
        bp.lcp_mvp(g, lam, out=w, gmres=gm)
    ms, its, fmm, dres, res = [], [], [], [], []
    for k in range(args.steps):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bp.contacts(g, cfg["delta"])
        _, st = bp.lcp_mvp(g, lam, out=w, gmres=gm)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
        its.append(st.iters)
        fmm.append(st.fmm_applies)
        dres.append(st.applies - st.fmm_applies)
        res.append(st.rel_resid)
    u = torch.empty((g.N, 3), dtype=torch.float64, device=dev)
    q = torch.tensor(np.random.default_rng(20264000).standard_normal((g.N, 3)), device=dev)
    bp.layer_apply(g, None, q, out=u)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    bp.layer_apply(g, None, q, out=u)
    e1.record(stream)
    torch.cuda.synchronize()
    out = {"ms_per_mvp": float(np.mean(ms)), "speedup_vs_direct_mvp": ms_direct / float(np.mean(ms)),
           "fmm_order": args.refine_order, "gmres_tol": args.gmres_tol, "fmm_krylov_steps_per_mvp": float(np.mean(fmm)),
           "direct_residuals_per_mvp": float(np.mean(dres)), "gmres_iters_per_mvp": float(np.mean(its)),
           "final_direct_rel_residual_max": float(np.max(res)),
           "mvp_rel_l2_vs_direct_mvp": float(torch.linalg.norm(w - w_ref) / torch.linalg.norm(w_ref)),
           "ms_fmm_layer_apply_d": e0.elapsed_time(e1), "geometry_init_s": round(t_init, 2),
           "timing": "CUDA events per MVP (contacts + MVP), L2 flushed between MVPs, %d MVPs" % args.steps}
    if not args.no_solve:
        pr, nr, gp = bp.contacts(g, cfg["delta"])
        meths = args.solvers.split(",")
        out["lcp_solve_bi"] = run_solve(args, cfg, g, pr, nr, gp, dev, meths[0], relax=True)
        for mth in meths[1:]:   # the other solvers with the same refined hi MVPs
            out["lcp_solve_" + mth] = run_solve(args, cfg, g, pr, nr, gp, dev, mth, relax=True)
    del g, u
    torch.cuda.empty_cache()
    return out


def run_fmm_large(args, dev, stream):
    """Context (an FMM for N >> 3e5): 4 096 unit spheres on a 16^3 lattice (the c4 recipe:
    spacing 2.02, jitter +-0.01) at the paper's p = 8, N = 589 824.  One D layer apply with the direct K1 and
    with the FMM far field (bpqn_disc_opts.fmm_order), their relative L2 difference, and one LCP MVP at
    GMRES 1e-8 in each mode (the FMM is an approximation; the direct sum is the north star's kernel)."""
    import torch
    import paper_2604_10089_b200 as bp
    rng = np.random.default_rng(20260099)
    n = 16
    g1 = np.arange(n) * 2.02
    C = np.array([[x, y, z] for x in g1 for y in g1 for z in g1]) + rng.uniform(-0.01, 0.01, (n ** 3, 3))
    q = None
    out = {"workload": "4096 spheres (16^3 lattice, spacing 2.02, jitter 0.01), p = 8", "fmm_order": args.fmm_order}
    ref = None
    for mode in ("direct", "fmm"):
        op = bp.default_disc_opts()
        op.fmm_order = args.fmm_order if mode == "fmm" else 0
        t0 = time.time()
        g = bp.Geometry(C, 8, opts=op)
        torch.cuda.synchronize()
        t_init = time.time() - t0
        if q is None:
            q = torch.tensor(rng.standard_normal((g.N, 3)), device=dev)
            out["N"] = g.N
        u = torch.empty((g.N, 3), dtype=torch.float64, device=dev)
        bp.layer_apply(g, None, q, out=u)
        ms = []
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            bp.layer_apply(g, None, q, out=u)
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        r = {"geometry_init_s": round(t_init, 2), "ms_layer_apply_d": float(np.median(ms))}
        if ref is None:
            ref = u.clone()
        else:
            r["rel_l2_vs_direct"] = float(torch.linalg.norm(u - ref) / torch.linalg.norm(ref))
        bp.contacts(g, 0.1)
        lam = torch.tensor(np.random.default_rng(20262099).uniform(0, 1, g.nc), device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        w, st = bp.lcp_mvp(g, lam, gmres=bp.default_gmres_opts(tol=1e-8))
        e1.record(stream)
        torch.cuda.synchronize()
        r.update({"contacts": g.nc, "ms_lcp_mvp": e0.elapsed_time(e1), "gmres_iters": st.iters})
        if mode == "direct":
            wref = w.clone()
        else:
            r["mvp_rel_l2_vs_direct"] = float(torch.linalg.norm(w - wref) / torch.linalg.norm(wref))
        out[mode] = r
        del g, u
        torch.cuda.empty_cache()
    out["speedup_layer_apply"] = out["direct"]["ms_layer_apply_d"] / out["fmm"]["ms_layer_apply_d"]
    out["speedup_mvp"] = out["direct"]["ms_lcp_mvp"] / out["fmm"]["ms_lcp_mvp"]
    return out


def run_c5(args, dev, stream):
    import torch
    import paper_2604_10089_b200 as bp
    from synth import layer_densities, make_config
    cfg = make_config(5)
    t0 = time.time()
    g = bp.Geometry(cfg["centers"], cfg["p"], cfg["radius"], cfg["mu"])
    torch.cuda.synchronize()
    t_init = time.time() - t0
    f_h, q_h = layer_densities(5, g.N)
    f = torch.tensor(f_h, device=dev)
    q = torch.tensor(q_h, device=dev)
    u = torch.empty((g.N, 3), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    for _ in range(2):
        bp.layer_apply(g, f, q, out=u)
    torch.cuda.synchronize()
    bp.profile_reset(g, events=True)
    ms = []
    for k in range(args.c5_steps):
        flush.fill_(float(k))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        bp.layer_apply(g, f, q, out=u)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    prof = bp.profile_get(g)
    m = float(np.mean(ms))
    k1_tflops = prof["allpairs_gflop"] / max(prof["ms_allpairs"], 1e-9)
    r = oracle_mvp_sample(cfg, 0, sd=True)     # the CPU oracle's S+D layer apply, sampled (bench.py model)
    out = {"workload": "c5 layer apply S+D (216 spheres, p=24, N=%d)" % g.N, "ms": m,
           "cpu_baseline": {"value": r["ms"], "unit": "ms", "cores": cores_used(), "kind": "oracle",
                            "sample": "far S+D sum for %d of %d targets (plain C, OpenMP) + near / self einsums, one "
                                      "application; host %s" % (r["n_targets"], r["N"], cpu_desc()),
                            "per_pass_s": r["per_pass_s"]},
           "pair_interactions_per_s": float(g.N) * g.N / (m * 1e-3),
           "k1_ms": prof["ms_allpairs"] / args.c5_steps, "k2_ms": prof["ms_near"] / args.c5_steps,
           "k3_ms": prof["ms_self"] / args.c5_steps,
           "k1_tflops": k1_tflops, "k1_frac_fp64_peak": k1_tflops / FP64_PEAK_TFLOPS,
           "near_incidences": g.n_incidences, "geometry_init_s": round(t_init, 3),
           "device_bytes": g.device_bytes}
    del g
    torch.cuda.empty_cache()
    return out


def main():
    args = parse()
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
