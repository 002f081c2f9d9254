#!/usr/bin/env python
"""Benchmark: walk-based Laplacian actions/s (𝕃·v, fp64) on BASELINE.json config C4.

Workload (N=1 and every N): config C4 — R-MAT n = 1e7, m = 2e8 (nnz 4e8), θ sweep
{0, 0.1, ..., 1} of the backtrack-downweighted Laplacian 𝕃_θ(exp(βx)), β = 1/ρ(A).
One step = 𝕃_θ v for all 11 θ (steps a3-a7, one batched Krylov action of 11 columns,
k = 30 Arnoldi steps on the companion operator Z); t_θ = φ_θ 1 (a8) is built once at operator
creation, outside the timed region (like the CSR upload a1).  Row-partitioned across N GPUs
(nnz-balanced), NCCL halo exchange + allreduce: strong scaling.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl walklap|reference] [--config c4]

Prints ONE JSON line (rank 0).  --impl reference times the CPU oracle (oracle/, fp64 series) on
the same workload, on the host cores, one action per step.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import graphgen as gg  # noqa: E402
from graphgen import configs  # noqa: E402

METRIC = "Laplacian actions/sec (L·v, fp64) and SpMV HBM GB/s vs peak"


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None

    def __enter__(self):
        self.first = ""
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", "200", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            # wait for the first sample: nvidia-smi's NVML start-up (driver calls, ~0.1-0.3 s) stays out of the
            # timed region (it delayed the host synchronisations of short steps, e.g. --rhoz: 201 -> 418 ms)
            self.first = self.p.stdout.readline()
        except Exception:
            self.p = None
        return self

    def __exit__(self, *exc):
        self.lines = []
        if self.p:
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                out = ""
            self.lines = [ln for ln in (self.first + (out or "")).splitlines() if ln.strip()]

    def summary(self):
        sm, smax, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(ngpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != ngpus and "WORLD_SIZE" in os.environ:
        raise SystemExit(f"--gpus {ngpus} but WORLD_SIZE={world}")
    return world, rank, local


def host_info() -> dict:
    """The host the CPU baseline ran on: CPU model, logical cores, BLAS threads."""
    model = None
    try:
        with open("/proc/cpuinfo") as fh:
            for ln in fh:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    blas = None
    try:
        from threadpoolctl import threadpool_info
        blas = [{"api": d.get("internal_api"), "threads": d.get("num_threads")} for d in threadpool_info()]
    except Exception:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "blas": blas}


def self_spawn(ngpus: int) -> int:
    """`bench.py --gpus N` without a launcher: start N ranks (one process per GPU) through
    torch.distributed.run on 127.0.0.1 with this same command line; rank 0 prints the JSON line."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={ngpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    log("self-spawn:", " ".join(cmd))
    return subprocess.call(cmd)


def load_graph(cfg, world, rank, torch, dist):
    """Rank 0 generates the seeded graph; N>1 broadcasts it over NCCL (setup, untimed)."""
    t0 = time.time()
    if rank == 0:
        g = cfg["make"]()
    if world > 1:
        meta = torch.tensor([g.n, g.nnz] if rank == 0 else [0, 0], dtype=torch.int64, device="cuda")
        dist.broadcast(meta, 0)
        n, nnz = int(meta[0]), int(meta[1])
        rp = torch.from_numpy(g.row_ptr).cuda() if rank == 0 else torch.empty(n + 1, dtype=torch.int64, device="cuda")
        ci = torch.from_numpy(g.col_idx).cuda() if rank == 0 else torch.empty(nnz, dtype=torch.int32, device="cuda")
        dist.broadcast(rp, 0)
        dist.broadcast(ci, 0)
        if rank != 0:
            g = gg.Graph(n, rp.cpu().numpy(), ci.cpu().numpy(), "broadcast")
        del rp, ci
    return g, time.time() - t0


def algorithmic_bytes(n, nnz, n_halo, G, K, Bmax, b, n_theta, reorth=2, esz=8, n_act=None):
    """Bytes each kernel must move per step, by kernel name.  esz: bytes per stored element of
    the TOAR batch's n-vectors (8; 4 in the fp32 mode, where the seeds, inputs and outputs stay double).
    n_act: the rows the Krylov vectors live on (wl_operator_active_rows: the isolated tail carries none); the
    inputs V, the outputs and t' cover all n rows."""
    n_out = n
    if n_act is not None and reorth == 2:
        n = n_act
    out = {}
    def add(k, v):
        out[k] = out.get(k, 0) + v
    for g0 in range(0, G, Bmax):
        B = min(Bmax, G - g0)
        L = 2 * n
        vec = 8 * L * B
        blk8 = 8 * n * B                 # a double n x B block (inputs, outputs, seeds)
        blk = esz * n * B                # a stored n x B block of the batch
        csr = 4 * nnz + 4 * (n + 1)
        if reorth == 2 and b < B and g0 % b == 0 and B % b == 0:
            bb = 8 * n * b                                              # θ-independent seeds over b columns
            add("spmv_binned", 2 * (csr + 2 * bb + 8 * n_halo * b))    # A v, A(Av)
            add("batch_inputs", 3 * bb + 2 * blk)                      # expand to the B columns
        else:
            add("spmv_binned", (csr + 2 * blk8 + 8 * n_halo * B))     # seed 1: gather y + write
            add("spmv_binned", (csr + 3 * blk8 + 8 * n_halo * B))     # seed 2: + x
        add("spmv_binned", K * (csr + 3 * blk + esz * n_halo * B))    # Z steps
        if reorth == 2:
            # TOAR: n-vector basis U (m = j+2 vectors at step j).  dots: Gram row of the newest U
            # vector + U^T y + |y|^2; update: u_m, x_{j+1}, z_{j+1} from y and U
            add("dcgs2_dots", 2 * blk)                                 # seed: (t0, b0)
            add("toar_update", 3 * blk)                                # seed: u_1
            for j in range(K):
                add("dcgs2_dots", (j + 3) * blk)
                add("toar_update", (j + 6) * blk)
            add("dcgs2_dots", (K + 2) * blk)                           # final Gram row
            add("combine", (K + 2) * blk + 8 * n_out * B + 8 * n_out * b + 8 * n_out * n_theta)
        else:
            # DCGS2 step j: dots read q_0..q_{j-1}, p_j and the SpMM output (w's top half IS p_j's
            # bottom half, read once); update reads the same and writes q_j and p_{j+1}
            for j in range(K):
                add("dcgs2_dots", (j + 1.5) * vec)
                add("dcgs2_update", (j + 3.5) * vec)
            add("dcgs2_dots", (K + 1) * vec)                          # final delayed reorth.
            add("combine", K * blk + blk + 8 * n * b + 8 * n * n_theta)
        add("batch_inputs", 8 * n * b + blk8)
    return out


def run_walklap(args):
    import torch
    import torch.distributed as dist
    import paper_2601_11338_b200 as wl

    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.get(args.config)
    g, t_gen = load_graph(cfg, world, rank, torch, dist)
    bounds = wl.partition(g.row_ptr, world)
    rb, re = int(bounds[rank]), int(bounds[rank + 1])
    rp = g.row_ptr[rb:re + 1]
    ci = g.col_idx[g.row_ptr[rb]:g.row_ptr[re]]
    comm = wl.Comm(rank, world, local) if world > 1 else None
    t0 = time.time()
    # β = 1/ρ(A) (inverse temperature) — ρ(A) by the library's Lanczos on A
    probe = wl.Operator(g.n, rp, ci, thetas=[1.0], f=("series", [0.0, 1.0]), row_range=(rb, re), comm=comm,
                        krylov_dim=2)
    # the Lanczos of ρ(A) runs rho_k single-column SpMVs A·y: time them live (b = 1 SpMV roofline)
    torch.cuda.synchronize()
    wl.profile_enable(True)
    rho = probe.spectral_radius(k=args.rho_k)
    wl.profile_enable(False)
    prof_rho = wl.profile_collect()
    spmv_b1 = None
    if "spmv_binned" in prof_rho:
        ms1, cnt1 = prof_rho["spmv_binned"]
        nl, nz = probe.n_local, probe.nnz_local
        by1 = 4 * nz + 4 * (nl + 1) + 8 * nl + 8 * probe.n_halo + 8 * nl  # col, rowptr, y (once), halo, out
        spmv_b1 = {"alg_bytes_per_launch": by1, "ms_per_launch": ms1 / cnt1, "launches": cnt1,
                   "achieved_gbs": by1 / (ms1 / cnt1 / 1e3) / 1e9}
        # per degree class when the library splits the launch scopes (WL_SPMV_SPLIT, profiling only)
        cls = {k: v[0] / cnt1 for k, v in prof_rho.items() if k.startswith("spmv_") and k != "spmv_binned"}
        if cls:
            spmv_b1["class_ms_per_launch"] = cls
    probe.close()
    beta = 1.0 / rho
    # --walk: the all-walk operator (θ = 1) on b = 11 input columns, the same B = 11 batch as the θ sweep:
    # Lanczos on A (opts.lanczos, default) against TOAR on Z (--lanczos 0) — the Gram bytes μ = 0 saves
    thetas = [1.0] if args.walk else cfg["thetas"]
    K = args.krylov if args.krylov else cfg["krylov_dim"]
    op = wl.Operator(g.n, rp, ci, thetas=thetas, f=("exp", beta), row_range=(rb, re), comm=comm, krylov_dim=K,
                     relabel=args.relabel, max_cols=args.max_cols,
                     krylov_tol=args.adaptive if args.adaptive > 0 else 0.0,
                     krylov_adaptive=1 if args.adaptive > 0 else 0, lanczos=args.lanczos, fp32=args.fp32)
    torch.cuda.synchronize()
    t_create = time.time() - t0
    b = args.b if args.b else (11 if args.walk else cfg["b"])
    n_loc = op.n_local
    Vfull = gg.vectors(g.n, b, cfg["vec_seed"] or 103)
    V = torch.from_numpy(np.ascontiguousarray(Vfull[rb:re])).cuda()
    del Vfull
    G = op.n_theta * b
    out = torch.empty((n_loc, G), dtype=torch.float64, device="cuda")
    ws = op.workspace(b)
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        op.apply(V, out=out, ws=ws)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = wl.launch_count()
    _, ks0, kb0 = ws.stats()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            op.apply(V, out=out, ws=ws)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = wl.launch_count() - l0
    _, ks1, kb1 = ws.stats()
    k_mean = (ks1 - ks0) / max(1, kb1 - kb0)
    ms = ev0.elapsed_time(ev1) / args.steps
    # per-kernel table: the same K steps again with per-launch-scope CUDA events (kept out of the timed region)
    torch.cuda.synchronize()
    wl.profile_enable(True)
    for _ in range(args.steps):
        op.apply(V, out=out, ws=ws)
    torch.cuda.synchronize()
    wl.profile_enable(False)
    prof = wl.profile_collect()
    graph_info = None
    if args.graph:
        # the whole step captured as one CUDA graph (no host synchronisation inside an action)
        cg = torch.cuda.CUDAGraph()
        with torch.cuda.graph(cg):
            op.apply(V, out=out, ws=ws)
        cg.replay()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            cg.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        gms = g0.elapsed_time(g1) / args.steps
        graph_info = {"ms_per_step": gms, "value": op.n_theta * b / (gms / 1e3)}
        del cg
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    actions = G  # every step applies 𝕃_θ to b vectors for each θ (whole job, all ranks together)
    value = actions / (ms / 1e3)

    # ---- end to end through the public C ABI with host buffers (pinned), H2D + D2H inside ----
    e2e = None
    if not args.no_e2e:
        Vh = torch.from_numpy(np.ascontiguousarray(V.cpu().numpy())).pin_memory().numpy()
        LVh = torch.empty((n_loc, G), dtype=torch.float64).pin_memory().numpy()
        op.apply_host(Vh, out=LVh, ws=ws)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        for _ in range(args.steps):
            op.apply_host(Vh, out=LVh, ws=ws)
        e_ms = (time.perf_counter() - t1) * 1e3 / args.steps
        if world > 1:
            t = torch.tensor([e_ms], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e_ms = float(t.item())
        e2e = {"value": actions / (e_ms / 1e3), "unit": "actions/s", "ms_per_step": e_ms,
               "h2d_bytes_per_step": int(Vh.nbytes) * world, "d2h_bytes_per_step": int(LVh.nbytes) * world}

    # ---- roofline of the dominant kernel (rank 0's kernels; live CUDA-event timing) ----
    peak, peak_src = peaks()
    nnz_loc = int(ci.shape[0])
    Kab = int(round(k_mean)) if args.adaptive > 0 else K  # the steps actually taken
    ab = algorithmic_bytes(n_loc, nnz_loc, op.n_halo, G, Kab, ws_bmax(op, b), b, op.n_theta, reorth=op.reorth,
                           esz=4 if args.fp32 else 8, n_act=op.n_active)
    if args.walk and args.lanczos:  # Lanczos batches (R19): K + 1 SpMMs (no diagonal term), 8 n-blocks per step
        na = op.n_active            # the Krylov vectors' rows (the isolated tail carries none)
        esz = 4 if args.fp32 else 8  # stored element of the Lanczos vectors (R21)
        blk, blk8 = esz * na * G, 8 * na * G
        csr = 4 * nnz_loc + 4 * (na + 1)
        ab = {"spmv_binned": (csr + 2 * blk8 + 8 * op.n_halo * G) + Kab * (csr + 2 * blk + esz * op.n_halo * G),
              "lanczos_vec": Kab * 8 * blk + 3 * blk,
              "combine": Kab * blk + 8 * n_loc * G + 8 * n_loc * b + 8 * n_loc, "batch_inputs": 8 * na * b + blk8}
    kernels = {}
    for name, (tot_ms, cnt) in prof.items():
        per_step_ms = tot_ms / args.steps
        bytes_ = ab.get(name)
        kernels[name] = {"ms_per_step": per_step_ms, "launches_per_step": cnt / args.steps,
                         "share": per_step_ms / ms}
        if bytes_:
            gbs = bytes_ / (per_step_ms / 1e3) / 1e9
            kernels[name].update({"alg_bytes_per_step": bytes_, "achieved_gbs": gbs, "frac": gbs / peak})
    top = max((k for k in kernels if "alg_bytes_per_step" in kernels[k]), key=lambda k: kernels[k]["ms_per_step"])
    headline = args.config == "c4" and not args.walk and not args.b and not args.krylov  # the captured workload
    ncu = ncu_traffic("f32" if args.fp32 else "f64") if headline else {}
    roof = {"kernel": top, "bound": "hbm", "achieved": kernels[top]["achieved_gbs"], "peak": peak,
            "unit": "GB/s", "frac": kernels[top]["frac"], "peak_source": peak_src,
            "traffic": ncu.get(top) if world == 1 else None,  # the committed ncu capture is single-GPU
            "alg_bytes_per_launch": ab[top] / max(1, kernels[top]["launches_per_step"])}
    if top == "spmv_binned" and ncu.get(top) and world == 1:
        # the SpMM's real bound is the rate HBM serves random rows: context for `frac`
        ms_launch = kernels[top]["ms_per_step"] / max(1, kernels[top]["launches_per_step"])
        roof["traffic_gbs"] = ncu[top] / (ms_launch / 1e3) / 1e9
        roof["traffic_frac"] = roof["traffic_gbs"] / peak
        roof["gathers_per_s"] = nnz_loc / (ms_launch / 1e3)
        if args.config == "c4" and G == 11:
            # tools/gather_ceiling.cu (profiles/r02_gather_ceiling.txt): 4e8 gathers of 11-column rows drawn from the
            # C4 degree distribution — 32-byte lanes at the 128-byte row stride: 2.81 ms; fp32 rows (2 lanes of 8
            # floats, 64-byte stride): 1.83 ms — the gather-only ceilings of this SpMM
            ceil_ms = 1.83 if args.fp32 else 2.81
            roof["gather_ceiling_ms"] = ceil_ms
            roof["frac_of_gather_ceiling"] = ceil_ms / ms_launch
    spmv = kernels.get("spmv_binned", {})

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(g, cfg, beta, args)

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "actions/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32-storage/f64-accumulate" if args.fp32 else "f64",
            "data": "synthetic (seeded R-MAT, graphgen)",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "n": g.n, "nnz": g.nnz,
                       "thetas": thetas, "b": b, "actions_per_step": actions, "krylov_dim": K,
                       "krylov_adaptive": ({"tol": args.adaptive, "mean_steps": k_mean} if args.adaptive > 0 else None),
                       "f": f"exp(beta x), beta=1/rho(A)={beta:.6g}", "global_batch": actions,
                       "parallelism": f"row-partition x{world} (NCCL halo + allreduce)",
                       "l2": "inputs larger than L2 (col_idx 1.6 GB, basis tens of GB): no flush",
                       "setup_s": {"generate": round(t_gen, 2), "operator_create_incl_t": round(t_create, 2)}},
            "roofline": roof,
            "spmv": {"b": G if G <= 32 else 32, "achieved_gbs": spmv.get("achieved_gbs"), "frac": spmv.get("frac"),
                     "peak": peak, "share": spmv.get("share"),
                     "traffic": ncu.get("spmv_binned") if world == 1 else None,
                     "b1": (dict(spmv_b1, frac=spmv_b1["achieved_gbs"] / peak) if spmv_b1 else None)},
            "kernels": {k: {kk: (round(vv, 6) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                        for k, v in sorted(kernels.items(), key=lambda kv: -kv[1]["ms_per_step"])},
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches, "clocks": clocks,
        }
        if graph_info:
            line["cuda_graph"] = graph_info
        print(json.dumps(line), flush=True)
    op.close()
    if comm:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def ws_bmax(op, b):
    return max(1, min(32, op.n_theta * b))


def ncu_traffic(mode="f64"):
    """DRAM bytes per launch of the C4 bench kernels from the committed ncu launch list (profiles/ncu_traffic.json,
    one table per storage mode: "f64" and "f32"), if present."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        tab = json.load(open(p)).get(mode, {})
        return {k: v["dram_bytes_per_launch"] for k, v in tab.items() if isinstance(v, dict)}
    except Exception:
        return {}


def _oracle_sample(g, cfg, beta):
    """Bounded oracle sample: one action 𝕃_θ v at θ = 0.5 by the fp64 series (t precomputed, untimed)."""
    from oracle import coeffs as C
    from oracle import series as S
    import threadpoolctl
    A = S.csr(g)
    f = C.exp(beta)
    rho = 1.0 / beta
    v = gg.vectors(g.n, 1, cfg["vec_seed"] or 103)[:, 0]
    t = S.total_communicability(g, 0.5, f, rho, A=A)
    with threadpoolctl.threadpool_limits(1):
        t0 = time.perf_counter()
        _ = t * v - S.phi_apply(g, 0.5, f, v, rho, A=A)
        dt = time.perf_counter() - t0
    return dt


def cpu_baseline(g, cfg, beta, args):
    dt = _oracle_sample(g, cfg, beta)
    return {"value": 1.0 / dt, "unit": "actions/s", "cores": 1, "kind": "oracle",
            "sample": "one action L_theta v at theta=0.5 on the full graph (fp64 series oracle, "
                      "scipy CSR SpMV, 1 thread; t precomputed outside the timing)",
            "seconds": dt, "host": host_info()}


def run_cg(args):
    """--solver cg: the paper's §5.3 workload on a config's graph — one resolvent NBT
    Laplacian action 𝕃_1((1-αx)^{-1}) v for each of 4 α log-spaced in [1e-3, 10^-1/2]/ρ, CG to a
    relative residual of 1e-9 (Jacobi preconditioner instead of the paper's AMG).  ρ(Z_1) from
    wl_spectral_radius_z scales α.  A step applies all four operators."""
    import torch
    import torch.distributed as dist
    import paper_2601_11338_b200 as wl

    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.get(args.config)
    g, t_gen = load_graph(cfg, world, rank, torch, dist)
    bounds = wl.partition(g.row_ptr, world)
    rb, re = int(bounds[rank]), int(bounds[rank + 1])
    rp = g.row_ptr[rb:re + 1]
    ci = g.col_idx[g.row_ptr[rb]:g.row_ptr[re]]
    comm = wl.Comm(rank, world, local) if world > 1 else None
    t0 = time.time()
    probe = wl.Operator(g.n, rp, ci, thetas=[0.0], f=("series", [0.0, 1.0]), row_range=(rb, re), comm=comm,
                        krylov_dim=2)
    rho = probe.spectral_radius_z(0, k=args.rho_k)  # ρ(Z_1) by Arnoldi on Z (NEXT-4), as §5.3 prescribes
    probe.close()
    alphas = [a / rho for a in np.logspace(-3, -0.5, 4)]
    ops = [wl.Operator(g.n, rp, ci, variant="nbt", f=("resolvent", a), row_range=(rb, re), comm=comm, relabel=args.relabel,
                       solver="cg", cg_tol=1e-9) for a in alphas]
    torch.cuda.synchronize()
    t_create = time.time() - t0
    b = args.b if args.b else 1
    Vfull = gg.vectors(g.n, b, cfg["vec_seed"] or 103)
    V = torch.from_numpy(np.ascontiguousarray(Vfull[rb:re])).cuda()
    del Vfull
    outs = [torch.empty((op.n_local, b), dtype=torch.float64, device="cuda") for op in ops]
    wss = [op.workspace(b) for op in ops]

    def step():
        for op, o, w in zip(ops, outs, wss):
            op.apply(V, out=o, ws=w)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    stream = torch.cuda.current_stream()
    l0 = wl.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = wl.launch_count() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    wl.profile_enable(True)
    it0 = sum(w.cg_iterations() for w in wss)
    for _ in range(args.steps):
        step()
    torch.cuda.synchronize()
    wl.profile_enable(False)
    prof = wl.profile_collect()
    cg_iters = (sum(w.cg_iterations() for w in wss) - it0) / args.steps  # executed iterations per step
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    actions = len(alphas) * b
    value = actions / (ms / 1e3)
    # algorithmic bytes: SpMM as in §7 (y once, x = y here: 2 n b reads + write); CG vector kernels:
    # init 4 blocks, each executed iteration dot 2 + update 6 + direction 3 blocks
    n_loc, nnz_loc = ops[0].n_local, int(ci.shape[0])
    blk = 8 * n_loc * b
    peak, peak_src = peaks()
    kernels = {}
    for name, (tot, cnt) in prof.items():
        per = tot / args.steps
        kernels[name] = {"ms_per_step": per, "launches_per_step": cnt / args.steps, "share": per / ms}
    if "spmv_binned" in kernels:
        k = kernels["spmv_binned"]
        by = cg_iters * (4 * nnz_loc + 4 * (n_loc + 1) + 2 * blk + 8 * ops[0].n_halo * b)
        k.update({"alg_bytes_per_step": by, "achieved_gbs": by / (k["ms_per_step"] / 1e3) / 1e9})
    if "cg_vec" in kernels:
        k = kernels["cg_vec"]
        inits = len(alphas)
        iters = cg_iters  # launches past convergence inside a check interval exit at once: not counted
        by = inits * 4 * blk + iters * 11 * blk
        k.update({"alg_bytes_per_step": by, "achieved_gbs": by / (k["ms_per_step"] / 1e3) / 1e9,
                  "cg_iterations_per_step": iters})
    for k in kernels.values():
        if "achieved_gbs" in k:
            k["frac"] = k["achieved_gbs"] / peak
    top = max((k for k in kernels if "alg_bytes_per_step" in kernels[k]), key=lambda k: kernels[k]["ms_per_step"])
    tk = kernels[top]
    roof = {"kernel": top, "bound": "hbm", "achieved": tk["achieved_gbs"], "peak": peak, "unit": "GB/s",
            "frac": tk["frac"], "peak_source": peak_src, "traffic": None,
            "alg_bytes_per_launch": tk["alg_bytes_per_step"] / max(1, tk["launches_per_step"])}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "actions/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded graphgen)",
            "config": {"workload": f"{args.config}: {cfg['desc']}; resolvent NBT Laplacian by PCG (Jacobi), "
                                   f"4 alpha log-spaced in [1e-3, 10^-0.5]/rho(Z_1), rel. tol 1e-9 (paper 5.3)",
                       "n": g.n, "nnz": g.nnz, "b": b, "alphas": alphas, "rho_Z1": rho,
                       "actions_per_step": actions, "parallelism": f"row-partition x{world}",
                       "setup_s": {"generate": round(t_gen, 2), "operators_incl_t": round(t_create, 2)}},
            "roofline": roof,
            "kernels": {k: {kk: (round(vv, 6) if isinstance(vv, float) else vv) for kk, vv in v.items()}
                        for k, v in sorted(kernels.items(), key=lambda kv: -kv[1]["ms_per_step"])},
            "cpu_baseline": None, "e2e": None, "gpu_launches": launches, "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    for op in ops:
        op.close()
    if comm:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def run_diffusion(args):
    """--diffusion: step a9 on a config with a τ sweep (C3: NBT diffusion exp(-τ𝕃)x0 for 90 τ in [0,100],
    k_out = 80, x0 = e_center), one full sweep per step.  Each outer Lanczos step is one inner 𝕃 action
    (k = 30 Krylov on Z), so the rate is reported as inner Laplacian actions/s and sweeps/s."""
    import torch
    import torch.distributed as dist
    import paper_2601_11338_b200 as wl

    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.get(args.config if args.config != "c4" else "c3")
    g, t_gen = load_graph(cfg, world, rank, torch, dist)
    bounds = wl.partition(g.row_ptr, world)
    rb, re = int(bounds[rank]), int(bounds[rank + 1])
    rp = g.row_ptr[rb:re + 1]
    ci = g.col_idx[g.row_ptr[rb]:g.row_ptr[re]]
    comm = wl.Comm(rank, world, local) if world > 1 else None
    t0 = time.time()
    probe = wl.Operator(g.n, rp, ci, thetas=[1.0], f=("series", [0.0, 1.0]), row_range=(rb, re), comm=comm,
                        krylov_dim=2)
    rho = probe.spectral_radius(k=args.rho_k)
    probe.close()
    op = wl.Operator(g.n, rp, ci, thetas=cfg["thetas"], f=("exp", 1.0 / rho), row_range=(rb, re), comm=comm,
                     relabel=args.relabel, krylov_dim=cfg["krylov_dim"],
                     krylov_tol=args.adaptive if args.adaptive > 0 else 0.0,
                     krylov_adaptive=1 if args.adaptive > 0 else 0, fp32=args.fp32)
    torch.cuda.synchronize()
    t_create = time.time() - t0
    kind, lo, hi, nt = cfg.get("taus", ("linspace", 0.0, 100.0, 90))
    taus = np.linspace(lo, hi, nt)
    k_out = cfg.get("k_out", 80)
    x0 = np.zeros(re - rb)
    c = g.n // 2
    if rb <= c < re:
        x0[c - rb] = 1.0
    x0 = torch.from_numpy(x0).cuda()
    out = torch.empty((op.n_local, nt), dtype=torch.float64, device="cuda")
    ws = op.workspace(1)
    for _ in range(args.warmup):
        op.diffuse(x0, taus, k_out=k_out, out=out, ws=ws)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    l0 = wl.launch_count()
    _, ks0, kb0 = ws.stats()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            op.diffuse(x0, taus, k_out=k_out, out=out, ws=ws)
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = wl.launch_count() - l0
    _, ks1, kb1 = ws.stats()
    k_mean = (ks1 - ks0) / max(1, kb1 - kb0)  # inner Arnoldi steps per action
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    actions = k_out  # inner 𝕃 applications per sweep
    wl.profile_enable(True)
    op.diffuse(x0, taus, k_out=k_out, out=out, ws=ws)
    torch.cuda.synchronize()
    wl.profile_enable(False)
    kernels = {k: {"ms_per_step": v[0], "launches_per_step": v[1], "share": v[0] / ms}
               for k, v in sorted(wl.profile_collect().items(), key=lambda kv: -kv[1][0])}
    # algorithmic bytes per sweep: k_out inner B = 1 actions of k' steps + the outer Arnoldi
    # (DCGS2 ring passes on n-vectors: dots read q_0..q_{j-1}, p_j, w; update also writes q_j, p_{j+1})
    # + the τ combine
    n_l = op.n_local
    ab = {}
    inner = algorithmic_bytes(n_l, int(ci.shape[0]), op.n_halo, 1, int(round(k_mean)), 1, 1, 1, reorth=op.reorth,
                              esz=4 if args.fp32 else 8, n_act=op.n_active)
    for kk, v in inner.items():
        ab[kk] = ab.get(kk, 0) + k_out * v
    for j in range(k_out):
        ab["dcgs2_dots"] = ab.get("dcgs2_dots", 0) + (j + 2) * 8 * n_l
        ab["dcgs2_update"] = ab.get("dcgs2_update", 0) + (j + 4) * 8 * n_l
    ab["dcgs2_dots"] += (k_out + 1) * 8 * n_l
    ab["lanczos_combine"] = 8 * n_l * (k_out + nt)
    peak, peak_src = peaks()
    for kk, v in kernels.items():
        if ab.get(kk):
            v["alg_bytes_per_step"] = ab[kk]
            v["achieved_gbs"] = ab[kk] / (v["ms_per_step"] / 1e3) / 1e9
            v["frac"] = v["achieved_gbs"] / peak
    top = max((kk for kk in kernels if "alg_bytes_per_step" in kernels[kk]), key=lambda kk: kernels[kk]["ms_per_step"])
    roof = {"kernel": top, "bound": "hbm", "achieved": kernels[top]["achieved_gbs"], "peak": peak, "unit": "GB/s",
            "frac": kernels[top]["frac"], "peak_source": peak_src, "traffic": None,
            "alg_bytes_per_launch": ab[top] / max(1, kernels[top]["launches_per_step"])}
    if rank == 0:
        line = {
            "metric": METRIC, "value": actions / (ms / 1e3), "unit": "actions/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f32-storage/f64-accumulate (inner actions)" if args.fp32 else "f64", "data": "synthetic (seeded graphgen)",
            "config": {"workload": f"{cfg['desc']}; diffusion exp(-tau L)x0 (step a9), {nt} tau in [{lo}, {hi}], "
                                   f"k_out={k_out}, inner k={cfg['krylov_dim']}, theta={cfg['thetas']}",
                       "n": g.n, "nnz": g.nnz, "sweeps_per_s": 1e3 / ms,
                       "krylov_adaptive": ({"tol": args.adaptive, "mean_steps": k_mean} if args.adaptive > 0 else None),
                       "setup_s": {"generate": round(t_gen, 2), "operator_create_incl_t": round(t_create, 2)}},
            "roofline": roof, "kernels": kernels, "cpu_baseline": None, "e2e": None, "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    op.close()
    if comm:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def run_trace(args):
    """--trace: NEXT-2, Alg. 1 XNysTrace-exp with poles at ∞ (reading R16) in the shape of Fig. 7:
    M = 30 Gaussian probes, 90 t-points, on the config's graph (default C3, NBT θ = 0, f = exp(βx), β = 1/ρ(A)).
    One step = the whole curve: k block Laplacian actions on M columns + block Gram–Schmidt + the host
    estimator.  Reported as p̂ curves/s and inner Laplacian column-actions/s."""
    import torch
    import torch.distributed as dist
    import paper_2601_11338_b200 as wl

    world, rank, local = dist_setup(args.gpus)
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = configs.get(args.config if args.config != "c4" else "c3")
    g, t_gen = load_graph(cfg, world, rank, torch, dist)
    bounds = wl.partition(g.row_ptr, world)
    rb, re = int(bounds[rank]), int(bounds[rank + 1])
    rp = g.row_ptr[rb:re + 1]
    ci = g.col_idx[g.row_ptr[rb]:g.row_ptr[re]]
    comm = wl.Comm(rank, world, local) if world > 1 else None
    probe = wl.Operator(g.n, rp, ci, thetas=[1.0], f=("series", [0.0, 1.0]), row_range=(rb, re), comm=comm,
                        krylov_dim=2)
    rho = probe.spectral_radius(k=args.rho_k)
    probe.close()
    op = wl.Operator(g.n, rp, ci, thetas=cfg["thetas"][:1], f=("exp", 1.0 / rho), row_range=(rb, re), comm=comm,
                     relabel=args.relabel, krylov_dim=cfg["krylov_dim"],
                     krylov_tol=args.adaptive if args.adaptive > 0 else 0.0,
                     krylov_adaptive=1 if args.adaptive > 0 else 0, fp32=args.fp32)
    M, k = args.trace_m, args.trace_k
    rational = args.trace_poles == "aaa"
    # Fig. 7: [0, t*] = [0, 100], 90 points, AAA poles, inner solves at 1e-6; the polynomial
    # (poles at ∞) variant keeps round 1's [0, 10] grid
    ts = np.linspace(0.0, 100.0 if rational else 10.0, 90)
    Om = torch.from_numpy(np.ascontiguousarray(gg.vectors(g.n, M, 2026)[rb:re])).cuda()
    ws = op.workspace(M)
    info = {}
    if rational:
        poles = wl.aaa_exp_poles(float(ts.max()) * op.laplacian_bound(0))  # Alg. 1 line 3

        def curve():
            p_, e_, inf_ = op.xnystrace_exp_rational(Om, ts, poles=poles, inner_tol=args.trace_inner_tol,
                                                     inner_maxit=2000, ws=ws)
            info.update(inf_)
            return p_, e_
    else:
        def curve():
            return op.xnystrace_exp(Om, ts, k, ws=ws)
    for _ in range(args.warmup):
        p, e = curve()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    stream = torch.cuda.current_stream()
    l0 = wl.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            p, e = curve()
        ev1.record(stream)
        torch.cuda.synchronize()
    launches = wl.launch_count() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        tt = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    wl.profile_enable(True)
    curve()
    torch.cuda.synchronize()
    wl.profile_enable(False)
    kernels = {kk: {"ms_per_step": v[0], "launches_per_step": v[1], "share": v[0] / ms}
               for kk, v in sorted(wl.profile_collect().items(), key=lambda kv: -kv[1][0])}
    # every batched Laplacian action of the curve ends in one combine launch: bytes = actions x one M-column action
    # of the Arnoldi steps actually taken (k' under --adaptive)
    nact = kernels.get("combine", {}).get("launches_per_step", 0)
    _, ks, kb = ws.stats()
    k_act = int(round(ks / kb)) if (args.adaptive > 0 and kb) else cfg["krylov_dim"]
    ab = {kk: nact * v for kk, v in algorithmic_bytes(op.n_local, int(ci.shape[0]), op.n_halo, M, k_act,
                                                       M, M, 1, reorth=op.reorth, esz=4 if args.fp32 else 8,
                                                       n_act=op.n_active).items()}
    peak, peak_src = peaks()
    roof = roofline_of(kernels, ab, peak, peak_src)
    if rank == 0:
        line = {
            "metric": "XNysTrace-exp return-probability curves/s", "value": 1e3 / ms, "unit": "curves/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32-storage/f64-accumulate (inner actions)" if args.fp32 else "f64",
            "data": "synthetic (seeded graphgen)",
            "config": {"workload": (f"{cfg['desc']}; Alg. 1 with {len(info['poles'])} AAA poles (+conjugates, +inf), "
                                    f"MINRES inner solves to {args.trace_inner_tol:g}, M={M} probes, 90 t in [0,100]"
                                    if rational else
                                    f"{cfg['desc']}; Alg. 1 (poles at inf), M={M} probes, k={k} blocks, 90 t in [0,10]")
                                   + f", theta={cfg['thetas'][0]}, inner Krylov k={cfg['krylov_dim']}"
                                   + (f" (adaptive, tol {args.adaptive:g})" if args.adaptive > 0 else ""),
                       "n": g.n, "nnz": g.nnz,
                       "poles": [[float(z.real), float(z.imag)] for z in info.get("poles", [])],
                       "inner_minres_iterations": info.get("inner_iters"),
                       "inner_krylov_steps": k_act,
                       "column_actions_per_s": (None if rational else k * M / (ms / 1e3)),
                       "p_hat": [round(float(x), 6) for x in p[::10]], "e_hat": [float(x) for x in e[::10]]},
            "roofline": roof, "kernels": kernels, "cpu_baseline": None, "e2e": None, "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    op.close()
    if comm:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def roofline_of(kernels, ab, peak, peak_src):
    """Attach algorithmic bytes / GB/s / fraction to the kernels with a byte count; the roofline object of the
    dominant one (HBM bound)."""
    for k, v in kernels.items():
        if ab.get(k):
            v["alg_bytes_per_step"] = ab[k]
            v["achieved_gbs"] = ab[k] / (v["ms_per_step"] / 1e3) / 1e9
            v["frac"] = v["achieved_gbs"] / peak
    tops = [k for k in kernels if "alg_bytes_per_step" in kernels[k]]
    if not tops:
        return None
    top = max(tops, key=lambda k: kernels[k]["ms_per_step"])
    return {"kernel": top, "bound": "hbm", "achieved": kernels[top]["achieved_gbs"], "peak": peak, "unit": "GB/s",
            "frac": kernels[top]["frac"], "peak_source": peak_src, "traffic": None,
            "alg_bytes_per_launch": ab[top] / max(1, kernels[top]["launches_per_step"])}


def run_extra(args):
    """--markov / --rhoz: measurement lines for NEXT-3 (one step = nsteps Markov steps p_{k+1} = p_k P on the
    config's graph at θ = 0.5, each one φ action of k = 30) and NEXT-4 (one step = ρ(Z_1) by 60 Arnoldi steps on
    the 2n companion operator).  1 GPU."""
    import torch
    import paper_2601_11338_b200 as wl

    cfg = configs.get(args.config)
    t0 = time.time()
    g = cfg["make"]()
    t_gen = time.time() - t0
    probe = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[1.0], f=("series", [0.0, 1.0]), krylov_dim=2)
    rho = probe.spectral_radius(k=args.rho_k)
    probe.close()
    stream = torch.cuda.current_stream()
    if args.markov:
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[0.5], f=("exp", 1.0 / rho), krylov_dim=30)
        p0 = torch.from_numpy(np.abs(gg.vectors(g.n, 1, 7)[:, 0])).cuda()
        p0 /= p0.sum()
        nsteps = 4
        out = torch.empty((g.n, nsteps), dtype=torch.float64, device="cuda")
        ws = op.workspace(1)
        fn = lambda: op.markov(p0, nsteps, out=out, ws=ws)  # noqa: E731
        unit, per_step, what = "markov steps/s", nsteps, f"{nsteps} Markov steps at theta=0.5 (eq:let_there_be_markov)"
    else:
        op = wl.Operator(g.n, g.row_ptr, g.col_idx, thetas=[0.0], f=("series", [0.0, 1.0]), krylov_dim=2)
        fn = lambda: op.spectral_radius_z(0, k=60)  # noqa: E731
        unit, per_step, what = "estimates/s", 1, "rho(Z_1) by 60 Arnoldi steps on the companion operator"
    for _ in range(args.warmup):
        fn()
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = wl.launch_count()
    with ClockSampler(0) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            fn()
        ev1.record(stream)
        torch.cuda.synchronize()
    ms = ev0.elapsed_time(ev1) / args.steps
    launches = wl.launch_count() - l0
    wl.profile_enable(True)
    fn()
    torch.cuda.synchronize()
    wl.profile_enable(False)
    kernels = {k: {"ms_per_step": v[0], "launches_per_step": v[1], "share": v[0] / ms}
               for k, v in sorted(wl.profile_collect().items(), key=lambda kv: -kv[1][0])}
    # algorithmic bytes per step: Markov = nsteps B = 1 actions (k = 30 TOAR) + the chain's vector
    # passes; ρ(Z) = 60 DCGS2 Arnoldi steps on 2n-vectors with one b = 1 SpMM each
    n, nnz = g.n, g.nnz
    if args.markov:
        ab = {k: nsteps * v for k, v in algorithmic_bytes(n, nnz, 0, 1, 30, 1, 1, 1, reorth=2).items()}
        ab["markov_vec"] = nsteps * (24 * n + 16 * n) + 16 * n
    else:
        L, ks = 2 * n, 60
        ab = {"spmv_binned": ks * (4 * nnz + 4 * (n + 1) + 3 * 8 * n), "dcgs2_dots": 0, "dcgs2_update": 0}
        for j in range(ks):
            ab["dcgs2_dots"] += (j + 2) * 8 * L
            ab["dcgs2_update"] += (j + 4) * 8 * L
        ab["dcgs2_dots"] += (ks + 1) * 8 * L
    peak, peak_src = peaks()
    roof = roofline_of(kernels, ab, peak, peak_src)
    line = {"metric": what, "value": per_step / (ms / 1e3), "unit": unit, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded graphgen)",
            "config": {"workload": f"{args.config}: {cfg['desc']}", "n": g.n, "nnz": g.nnz, "rho_A": rho,
                       "setup_s": {"generate": round(t_gen, 2)}},
            "roofline": roof, "kernels": kernels, "gpu_launches": launches, "clocks": clk.summary()}
    if not args.markov:
        line["config"]["rho_Z1"] = op.spectral_radius_z(0, k=60)
    print(json.dumps(line), flush=True)
    op.close()


def run_reference(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = configs.get(args.config)
    g = cfg["make"]()
    from oracle import series as S
    rho = S.rho_A(g)
    beta = 1.0 / rho
    for _ in range(args.warmup):
        _oracle_sample(g, cfg, beta)
    times = [_oracle_sample(g, cfg, beta) for _ in range(args.steps)]
    ms = 1e3 * sum(times) / len(times)
    value = 1e3 / ms
    sample = ("one action L_theta v at theta=0.5 per step on the full graph (fp64 series oracle, "
              "scipy CSR SpMV, 1 thread; t precomputed outside the timing)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": "actions/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded R-MAT, graphgen)",
        "config": {"workload": f"{args.config}: {cfg['desc']}", "n": g.n, "nnz": g.nnz,
                   "f": f"exp(beta x), beta=1/rho(A)={beta:.6g}"},
        "cpu_baseline": {"value": value, "unit": "actions/s", "cores": 1, "kind": "oracle", "sample": sample,
                         "host": host_info()},
        "e2e": {"value": value, "unit": "actions/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="walklap", choices=["walklap", "reference"])
    ap.add_argument("--config", default="c4")
    ap.add_argument("--b", type=int, default=0)
    ap.add_argument("--krylov", type=int, default=0)
    ap.add_argument("--rho-k", type=int, default=60)
    ap.add_argument("--max-cols", type=int, default=32, help="columns per internal Krylov batch (opts.max_cols)")
    ap.add_argument("--walk", action="store_true", help="theta = 1 only, b = 11 columns (the mu = 0 Lanczos path)")
    ap.add_argument("--lanczos", type=int, default=1, choices=[0, 1], help="opts.lanczos (theta = 1 batches)")
    ap.add_argument("--adaptive", type=float, default=0.0,
                    help="> 0: stop each Arnoldi process once the a-posteriori estimate is below this (opts.krylov_adaptive)")
    ap.add_argument("--fp32", type=int, default=0, choices=[0, 1],
                    help="opts.fp32: float storage of the Krylov batches, double sums (parity 1e-4)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", action="store_true", help="also time the step captured as one CUDA graph")
    ap.add_argument("--diffusion", action="store_true", help="step a9: a full diffusion sweep (default config c3)")
    ap.add_argument("--markov", action="store_true", help="NEXT-3: Markov chain steps")
    ap.add_argument("--relabel", type=int, default=1, choices=[0, 1],
                    help="degree-sorted row relabelling inside the operator (opts.relabel)")
    ap.add_argument("--trace", action="store_true", help="NEXT-2: XNysTrace-exp return-probability curve")
    ap.add_argument("--trace-m", type=int, default=30, help="--trace: probes M")
    ap.add_argument("--trace-k", type=int, default=8, help="--trace: block Krylov steps k (poles at inf)")
    ap.add_argument("--trace-poles", default="aaa", choices=["aaa", "inf"],
                    help="--trace: AAA poles + MINRES shifted solves (Alg. 1 as in the paper) or all poles at inf")
    ap.add_argument("--trace-inner-tol", type=float, default=1e-6, help="--trace: MINRES relative tolerance (P:1483)")
    ap.add_argument("--rhoz", action="store_true", help="NEXT-4: rho(Z_1) by Arnoldi on the companion operator")
    ap.add_argument("--solver", default="krylov", choices=["krylov", "cg"],
                    help="cg: the paper's 5.3 resolvent workload by PCG on --config's graph")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl != "reference":
        raise SystemExit(self_spawn(args.gpus))
    if args.warmup < 3:
        log("warning: contract requires >= 3 warm-up steps")
    if args.impl == "reference":
        run_reference(args)
    elif args.solver == "cg":
        run_cg(args)
    elif args.trace:
        run_trace(args)
    elif args.diffusion:
        run_diffusion(args)
    elif args.markov or args.rhoz:
        run_extra(args)
    else:
        run_walklap(args)


if __name__ == "__main__":
    main()
