#!/usr/bin/env python
"""Benchmark: Chebyshev s-step PCG outer iterations with nu-sweep FGS Gram
solves on B200 (BASELINE.json metric: time per outer iteration and GDOF/s at
1/2/4/8 GPUs; fraction of the HBM roofline).

Workload (BASELINE.json configs[4], "cfg5"): 3D 7-point Poisson, 448^3
unknowns per GPU stacked in z (weak scaling, ~90M unknowns per GPU), FP64,
Jacobi, b ~ U[-1,1] (SplitMix64 on the global index, seed 42), x0 = 0,
analytic global spectral bounds, s = 16, nu = 30.  One "step" = one outer
iteration: s basis SpMVs (+halo exchange), the fused Gram pass + the single
allreduce, the FGS solve and the update.  Each step streams ~68 vectors of
0.72 GB (the basis P, w_{s-1}, x: ~13 GB touched per GPU, ~100x the 126 MB
L2), so no flush is needed between steps.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)
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

K1_NAME = "k1t"   # dominant kernel (basis step) as named in the ncu capture

# BASELINE.json configs (synthetic, seeded).  cfg5 is the
# configuration the headline metric is quoted on; the others are parity-test
# cases that bench.py can also time (--workload) for the per-kernel rooflines.
WORKLOADS = {
    "cfg1": {"kind": "5pt", "n": 64, "s": 8, "nu": 20, "bounds": "analytic",
             "desc": "cfg1: 2D 5-point Poisson {n}x{n} (n=4096), FP64, Jacobi, analytic bounds; latency: "
                     "microseconds per outer iteration under CUDA-graph replay (SURVEY 8(d))"},
    "cfg2": {"kind": "7pt", "n": 128, "s": 16, "nu": 25, "bounds": "analytic",
             "desc": "cfg2: 3D 7-point Poisson {n}^3 per GPU, FP64, Jacobi, analytic bounds"},
    "cfg3": {"kind": "27pt", "n": 256, "s": 16, "nu": 30, "bounds": "lanczos",
             "desc": "cfg3: 3D 27-point stencil {n}^3 per GPU (z-slab weak scaling), FP64, Jacobi, "
                     "Lanczos-50 bounds widened 5% (GPU, sscg_estimate_bounds)"},
    "cfg4": {"kind": "varcoef7", "n": 192, "s": 16, "nu": 30, "bounds": "lanczos",
             "desc": "cfg4: 3D variable-coefficient 7-point diffusion {n}^3 (lognormal faces, seed 42), FP64, "
                     "Jacobi, Lanczos-50 bounds widened 5% (GPU)"},
    "cfg5": {"kind": "7pt", "n": 448, "s": 16, "nu": 30, "bounds": "analytic",
             "desc": "cfg5: 3D 7-point Poisson {n}^3 per GPU (z-slab weak scaling), FP64, Jacobi, analytic bounds"},
    # not a BASELINE config: the general sparse path (SSCG_OP_CSR) on cfg 2's operator, assembled
    "csr": {"kind": "csr7", "n": 128, "s": 16, "nu": 25, "bounds": "analytic",
            "desc": "csr: the 3D 7-point Poisson operator {n}^3 assembled as CSR (general sparse path, one slab "
                    "per GPU; replicas for N > 1), FP64, Jacobi, analytic bounds"},
}
METRIC = "s-step CG time/outer-iter & GDOF/s at 1/2/4/8 B200; % of HBM peak"
UNIT = "GDOF/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)   # BASELINE cfg 5: "50 outer iterations timed"
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="cfg5", choices=sorted(WORKLOADS),
                    help="BASELINE.json config (default cfg5 = the headline metric's configuration)")
    ap.add_argument("--n", type=int, default=None, help="grid edge per GPU (default: the workload's)")
    ap.add_argument("--s", type=int, default=None)
    ap.add_argument("--nu", type=int, default=None)
    ap.add_argument("--strong", action="store_true", help="cfg4 (ii): fixed global n^3 split over the GPUs")
    ap.add_argument("--cpu-planes", type=int, default=16, help="z-planes of the oracle's CPU sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--gram-solver", default="fgs", choices=["fgs", "cholesky"],
                    help="K4: nu FGS sweeps (the paper's method, default) or the exact Cholesky solve (NEXT-2)")
    ap.add_argument("--block", action="store_true",
                    help="block-conjugate s-step CG (NEXT-2, DESIGN.md R24) instead of the restart form")
    a = ap.parse_args()
    w = WORKLOADS[a.workload]
    a.n = w["n"] if a.n is None else a.n
    a.s = w["s"] if a.s is None else a.s
    a.nu = w["nu"] if a.nu is None else a.nu
    a.kind = w["kind"]
    return a


def workload(a, nranks):
    n = a.n
    if a.kind == "5pt":   # 2D: one n x n grid per GPU (cfg 1 stays on one GPU; N > 1 runs replicas)
        return {"workload": WORKLOADS[a.workload]["desc"].format(n=n) + f", s={a.s}, nu={a.nu}, x0=0, "
                "b~U[-1,1] seed 42", "nx": n, "ny": n, "nz_per_gpu": 1, "nz_global": 1, "s": a.s, "nu": a.nu,
                "n_global": n * n * nranks, "parallelism": f"replicas x{nranks}" if nranks > 1 else "single GPU",
                "l2": "working set (%.2f MB) resident in the 126 MB L2: a latency measurement, no roofline claim"
                      % ((2 * a.s + 2) * n * n * 8 / 1e6)}
    csr = a.kind == "csr7"
    nzg = n if (a.strong or csr) else n * nranks
    desc = WORKLOADS[a.workload]["desc"].format(n=n)
    if a.strong:
        desc = desc.replace("per GPU", "global (strong scaling)")
    if a.block or a.gram_solver != "fgs":
        desc += "; variant: %s%s" % ("block-conjugate s-step CG, " if a.block else "", a.gram_solver + " Gram solve")
    if csr:
        return {"workload": f"{desc}, s={a.s}, nu={a.nu}, x0=0, b~U[-1,1] seed 42", "nx": n, "ny": n,
                "nz_per_gpu": n, "nz_global": n, "s": a.s, "nu": a.nu, "n_global": n * n * n * nranks,
                "parallelism": f"replicas x{nranks}" if nranks > 1 else "single GPU",
                "l2": "no flush: the matrix and s+2 vectors (%.2f GB) >> 126 MB L2" % ((a.s + 2 + 12) * n ** 3 * 8 / 1e9)}
    return {"workload": f"{desc}, s={a.s}, nu={a.nu}, x0=0, b~U[-1,1] seed 42",
            "nx": n, "ny": n, "nz_per_gpu": nzg // nranks, "nz_global": nzg, "s": a.s, "nu": a.nu,
            "n_global": n * n * nzg, "parallelism": f"z-slab x{nranks}",
            "l2": "no flush: per-GPU working set >= s+2 vectors (%.2f GB: basis, w_{s-1}, x) >> 126 MB L2"
                  % ((a.s + 2) * n * n * (nzg // nranks) * 8 / 1e9)}


# --------------------------------------------------------------------------
# CPU oracle (the reported baseline / --impl reference arm)
def oracle_sample(a, steps, warmup, planes=None):
    """Time `steps` outer iterations of the CPU oracle on a bounded sample:
    the first `cpu_planes` z-planes of the same n x n grid (Dirichlet box of
    n x n x cpu_planes, same s, nu, seed; bounds of that box).  Returns
    (GDOF/s, seconds per step, description)."""
    import inputs
    import oracle as orc
    n, zs = a.n, min(planes or a.cpu_planes, a.n)
    if a.kind == "5pt":
        zs = 1
    b = inputs.rhs_uniform(n, n, zs, seed=42)
    if a.kind == "5pt":
        A = orc.stencil(orc.KIND_5PT2D, n, n, 1)
        lmin, lmax = inputs.analytic_bounds("5pt", n, n)
    elif a.kind == "varcoef7":
        A = orc.stencil(orc.KIND_VARCOEF7, n, n, zs, *inputs.lognormal_faces(n, n, zs, seed=42))
        lmin, lmax, _ = orc.lanczos_bounds(A, 50, b, 0.05)     # untimed setup
    elif a.kind == "csr7":   # the oracle's CSR operator on the sample
        A = orc.csr(*inputs.stencil7_csr_fast(n, n, zs))
        lmin, lmax = inputs.analytic_bounds("7pt", n, n, zs)
    else:
        A = orc.stencil({"7pt": orc.KIND_7PT, "27pt": orc.KIND_27PT}[a.kind], n, n, zs)
        lmin, lmax = inputs.analytic_bounds(a.kind, n, n, zs)
    t0 = time.perf_counter()
    orc.sstep_cg(A, lmin, lmax, a.s, a.nu, b, rtol=0.0, max_outer=warmup)
    t1 = time.perf_counter()
    orc.sstep_cg(A, lmin, lmax, a.s, a.nu, b, rtol=0.0, max_outer=warmup + steps)
    t2 = time.perf_counter()
    per = ((t2 - t1) - (t1 - t0)) / steps
    if per <= 0.0:   # tiny samples: the difference drowns in setup noise
        per = (t2 - t1) / (warmup + steps)
    npts = n * n * zs
    desc = (f"oracle/sscg_oracle.c (gcc -O2 -fopenmp, FP64), {a.kind}, on a {n}x{n}x{zs} sample "
            f"({npts} unknowns), {steps} outer iterations timed as t(max_outer={warmup + steps}) - "
            f"t(max_outer={warmup})")
    return npts / per / 1e9, per, desc


def host_info():
    """MemTotal / MemAvailable and a host copy-bandwidth probe (numpy copy of
    a 1 GiB array, best of 3; read + write bytes) -- SURVEY 8(d) asks for both
    beside the oracle baseline."""
    import numpy as np
    info = {}
    try:
        for line in open("/proc/meminfo"):
            k, v = line.split(":", 1)
            if k in ("MemTotal", "MemAvailable"):
                info[k + "_GB"] = round(int(v.split()[0]) / 2 ** 20, 1)
    except OSError:
        pass
    try:
        src = np.ones(1 << 27)   # 1 GiB
        dst = np.empty_like(src)
        best = None
        for _ in range(3):
            t0 = time.perf_counter()
            np.copyto(dst, src)
            dt = time.perf_counter() - t0
            best = dt if best is None else min(best, dt)
        info["host_copy_gbs"] = round(2 * src.nbytes / best / 1e9, 2)
        info["host_copy_note"] = "numpy copy of 1 GiB, one thread, best of 3 (read + write bytes)"
    except MemoryError:
        pass
    return info


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def cpu_model():
    """The host CPU the oracle baseline ran on (report the CPU model)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(a):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    value, per, desc = oracle_sample(a, a.steps, a.warmup)
    cfg = workload(a, a.gpus)
    if a.kind == "5pt":
        cfg["us_per_outer"] = per * 1e6
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": per * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference", "config": cfg,
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle", "sample": desc,
                             "cpu": cpu_model()},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampler (B200_PROFILING.md): started before the warm-up so the
    tool is already emitting when the timed region begins; samples whose
    timestamps fall in the timed region are summarised (all samples under load
    if the region is shorter than the 100 ms sampling interval)."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap,power.draw,power.limit,clocks.mem")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.p = None
        self.t0 = self.t1 = None
        self.out = ""

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.gpu), "-lms", "100"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def begin(self):
        self.t0 = time.time()

    def end(self):
        self.t1 = time.time()

    def stop(self):
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        import datetime
        rows = []
        for line in (self.out or "").splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f").timestamp()
            except ValueError:
                ts = None
            rows.append((ts, f[1:]))
        window = "timed region"
        sel = [r for ts, r in rows if ts is not None and self.t0 is not None and self.t0 - 0.05 <= ts <= self.t1 + 0.05]
        if not sel:
            sel, window = [r for _, r in rows], "warm-up + timed region"
        sm, mx, reasons, pw, pl, mem = [], [], set(), [], [], []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for f in sel:
            try:
                sm.append(float(f[1])); mx.append(float(f[2]))
            except (ValueError, IndexError):
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
            for lst, k in ((pw, 8), (pl, 9), (mem, 10)):   # informational: power and memory clock
                try:
                    lst.append(float(f[k]))
                except (ValueError, IndexError):
                    pass
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        out = {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
               "samples": len(sm), "window": window}
        if pw:
            out["power_w"] = statistics.median(pw)
        if pl:
            out["power_limit_w"] = max(pl)
        if mem:
            out["mem_mhz"] = statistics.median(mem)
        return out


def max_over_ranks(dist, v: float, device="cuda") -> float:
    """Max of a per-rank time over all ranks (dist = torch.distributed or None)."""
    if dist is None:
        return v
    import torch
    t = torch.tensor([v], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def ncu_traffic(n, kernel_prefix):
    """dram bytes (read + write) per launch of the dominant kernel from the
    latest committed `ncu --set full` capture of this workload
    (profiles/r*_ncu_full_<n>.json, written by tools/ncu_raw_summary.py), else
    None.  The capture is of the same bench command (one launch)."""
    import glob
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_full_%d.json" % n)), reverse=True):
        try:
            d = json.load(open(f))
        except Exception:
            continue
        for name, rec in d.items():
            if name.startswith(kernel_prefix):
                rd, wr = rec["dram__bytes_read.sum"], rec["dram__bytes_write.sum"]
                return rd[0] * scale.get(rd[1], 1.0) + wr[0] * scale.get(wr[1], 1.0)
    return None


def mix_ceiling(reads, writes):
    """Measured HBM ceiling (GB/s) of a plain streaming kernel with this
    read:write vector mix (tools/membw.cu, committed under profiles/), or None."""
    import glob
    import re
    for f in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_membw_mix_ceilings.txt")), reverse=True):
        for line in open(f):
            m = re.match(r"R=\s*(\d+) W=(\d+)\s+[\d.]+ ms\s+([\d.]+) GB/s", line.strip())
            if m and int(m.group(1)) == reads and int(m.group(2)) == writes:
                return float(m.group(3)), os.path.basename(f)
    return None, None


def run_ours(a):
    import numpy as np
    import torch

    import inputs
    import paper_2512_09642_b200 as sscg

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus:
        raise SystemExit(f"--gpus {a.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    n, s, nu = a.n, a.s, a.nu
    twod = a.kind == "5pt"          # cfg 1: one 2D grid per GPU (replicas for N > 1)
    csr = a.kind == "csr7"          # the general sparse path: one slab per process (replicas for N > 1)
    replica = twod or csr
    nz = 1 if twod else (n if (a.strong or csr) else n * world)
    z0, nzl = (0, 1) if twod else (0, nz) if csr else sscg.partition(nz, world, 1, rank)
    b_host = torch.from_numpy(inputs.rhs_uniform(n, n, nz, seed=42, z0=z0, nzl=nzl)).pin_memory()
    b = b_host.cuda()
    nid = None
    if world > 1 and not replica:
        obj = [sscg.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    faces = None
    if a.kind == "varcoef7":
        kx, ky, kz = inputs.lognormal_faces(n, n, nz, seed=42)
        faces = [torch.from_numpy(np.ascontiguousarray(f)).cuda()
                 for f in (kx[z0:z0 + nzl], ky[z0:z0 + nzl], kz[z0:z0 + nzl + 1])]
        del kx, ky, kz
        op = sscg.Stencil("varcoef7", n, n, nz, *faces)
    elif csr:
        csr_arrays = [torch.from_numpy(v).cuda() for v in inputs.stencil7_csr_fast(n, n, nz)]
        op = sscg.CSR(*csr_arrays)
    else:
        op = sscg.Stencil(a.kind, n, n, nz)
    variant = {"gram_solver": a.gram_solver, "block": a.block}
    if twod:
        S = sscg.Solver(op, *inputs.analytic_bounds(a.kind, n, n), s, nu, **variant)
    elif csr:
        S = sscg.Solver(op, *inputs.analytic_bounds("7pt", n, n, nz), s, nu, **variant)
    elif WORKLOADS[a.workload]["bounds"] == "analytic":
        S = sscg.Solver(op, *inputs.analytic_bounds(a.kind, n, n, nz), s, nu, rank=rank, nranks=world, nccl_id=nid,
                        **variant)
    else:   # 50 Lanczos steps on the GPU, widened 5 % (R13), untimed setup
        S = sscg.Solver(op, 0.0, 0.0, s, nu, rank=rank, nranks=world, nccl_id=nid, **variant)
        S.set_bounds(*S.estimate_bounds(b, 50, 0.05))
    n_local, n_global = S.n_local, n * n * nz * (world if replica else 1)

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    # r_0 = b and the first basis/Gram (untimed), then W warm-up steps
    clk = Clocks(local).start()
    x = S.solve(b, rtol=0.0, max_outer=0)
    S.iterate(x, a.warmup)
    # timed region: exactly K outer iterations (CUDA-graph replay), device-timed
    # inside the library with CUDA events on its stream
    barrier()
    clk.begin()
    S.iterate(x, a.steps)
    barrier()
    clk.end()
    clk.stop()
    st = S.stats()
    ms = max_over_ranks(dist, st.ms_total)
    value = n_global * a.steps / (ms / 1e3) / 1e9
    launches = st.kernel_launches
    # second pass of the same K steps with every launch bracketed by events
    # (per-kernel times for the roofline; plain launches, no graph)
    barrier()
    S.set_profiling(True)
    S.iterate(x, a.steps)
    barrier()
    st_prof = S.stats()
    prof = S.profile()
    S.set_profiling(False)

    # roofline of the dominant kernel (K1: basis step) and the others
    peak, peak_src = peaks()
    vec = 8.0 * n_local
    face_bytes = 0.0
    if a.kind == "varcoef7":   # kx, ky, kz of this slab, read by every basis step
        face_bytes = 8.0 * (n * (n + 1) * S.nz_local * 2 + n * n * (S.nz_local + 1))
    if csr:                    # the matrix, streamed by every SpMV: rowptr (8 B/row), colind + val (12 B/nnz)
        face_bytes = 8.0 * (n_local + 1) + 12.0 * float(csr_arrays[1].numel())
    basis_vecs = S.query(sscg.QUERY_BASIS_VECTORS)       # (4s-3) single steps, fewer with pairs / triples
    single_vecs = S.query(sscg.QUERY_BASIS_SINGLE_VECTORS)   # the single steps of a fused schedule (j = s-1)
    depth = S.query(sscg.QUERY_BASIS_FUSED)               # basis steps per launch: 1, 2 (K1F) or 3 (K1M)
    fused = depth > 1
    upd_vecs = S.query(sscg.QUERY_UPDATE_VECTORS)        # 2s+3, or s+4 with W alpha from the recurrence
    gram_vecs = S.query(sscg.QUERY_GRAM_VECTORS)         # 2s, or s+1 with W recovered from the recurrence
    face_passes = s if depth == 1 else (s + 1) // 2   # fused pairs read the faces once per pair
    # "basis": the fused basis launches (K1M triples / K1F pairs) -- the dominant
    # kernel; "basis_single": the single steps around them (the last step j = s-1)
    bytes_per_outer = {"basis": (basis_vecs - single_vecs) * vec + face_passes * face_bytes,
                       "basis_single": single_vecs * vec, "gram": gram_vecs * vec, "update": upd_vecs * vec}
    kern = {}
    for k, byt in bytes_per_outer.items():
        t_ms, cnt = prof[k]
        if cnt == 0:
            continue
        per_launch = byt * a.steps / max(cnt, 1)
        gbs = per_launch / (t_ms / max(cnt, 1) / 1e3) / 1e9 if t_ms > 0 else None
        kern[k] = {"launches": cnt, "ms_per_launch": t_ms / max(cnt, 1), "bytes_per_launch": per_launch,
                   "achieved_gbs": gbs, "frac": (gbs / peak) if gbs else None,
                   "share_of_step": t_ms / st_prof.ms_total if st_prof.ms_total else None}
    # the Gram pass also against the FP64 pipe (the limit at s >= 24): FP64 issue slots
    # per grid point of the kernel as launched -- the tensor-core pass (K2R / K2D, s > 8 or the folded
    # schedule) forms every 8 x 8 tile of a block triangle of ceil(s/8) blocks by DMMA m8n8k4 (64 FMA
    # per tile and point) and c_i = p_i^T p_0 by s FMAs; the streaming pass K2S (s <= 8) forms
    # s(s+1)/2 + s entries by DFMA; the W-free passes add 3 FP64 operations per recovered w_j(point).
    # Peak: the DMMA rate measured by tools/dmma_probe.cu (profiles/r02a_dmma_probe.txt, 37.1 TFLOP/s
    # = 18.55e12 FMA/s; DFMA alone measured 33.9).
    if "gram" in kern and kern["gram"]["ms_per_launch"] > 0 and not csr:
        wfree_g = gram_vecs < 2 * s
        nb = (s + 7) // 8
        if wfree_g:   # K2S for s <= 8 unless SSCG_K2S=0, else K2R
            tensor = s > 8 or os.environ.get("SSCG_K2S", "1") == "0"
        else:         # stored W: K2D for s > 16 unless forced, else the register-tiled K2
            tensor = os.environ.get("SSCG_K2_DMMA", "1" if s > 16 else "0") == "1"
        fma_pt = (64 * nb * (nb + 1) // 2 + s) if tensor else (s * (s + 1) // 2 + s)
        if wfree_g:
            fma_pt += 3 * s
        gl = kern["gram"]
        fma_s = fma_pt * (n_local * a.steps / max(gl["launches"], 1)) / (gl["ms_per_launch"] / 1e3)   # points per launch
        gl["fp64_pipe"] = {"fma_slots_per_point": fma_pt, "achieved_tflops": 2 * fma_s / 1e12,
                           "peak_tflops": 37.1, "frac": 2 * fma_s / 1e12 / 37.1,
                           "peak_source": "profiles/r02a_dmma_probe.txt (FP64 DMMA, 8-16 warps per SM)",
                           "kernel": ("K2R" if wfree_g else "K2D/K2") if tensor else "K2S"}
    for k in ("fgs", "allreduce", "halo"):
        t_ms, cnt = prof[k]
        kern[k] = {"launches": cnt, "us_per_launch": 1e3 * t_ms / max(cnt, 1),
                   "share_of_step": t_ms / st_prof.ms_total if st_prof.ms_total else None}
    kern["profiled_pass_ms_per_step"] = st_prof.ms_total / a.steps
    k1 = kern["basis"]
    path_bytes = sum(bytes_per_outer.values())
    cfg = workload(a, world)
    k1_name = {3: "k1m", 2: "k1f"}.get(depth, "k1_csr" if csr else K1_NAME)
    # read : write vectors of one interior basis launch (W recovered in the Gram pass: p only)
    wfree = gram_vecs < 2 * s
    mixrw = (2, depth) if wfree else (2, 2 * depth)
    mc = mix_ceiling(*mixrw)
    roof = {"bound": "hbm", "kernel": "K1 %s<%s> (%sSpMV + Jacobi + Chebyshev recurrence)"
                                      % (k1_name, a.kind, {3: "three basis steps per launch: ",
                                                           2: "two basis steps per launch: "}.get(depth, "")),
            "achieved": k1["achieved_gbs"], "peak": peak, "unit": "GB/s", "frac": k1["frac"],
            "traffic": ncu_traffic(n, k1_name) if a.workload == "cfg5" else None, "peak_source": peak_src,
            "traffic_note": "ncu dram read+write of one interior launch (algorithmic: %d vectors = %.4g B)"
                            % (sum(mixrw), sum(mixrw) * vec),
            "bytes_rule": "%d FP64 vectors per outer in the %s (+ s face sets for varcoef7), / their launches; "
                          "path: + %d (single basis steps) + %d (Gram) + %d (update) vectors"
                          % (basis_vecs - single_vecs, {3: "K1M triples", 2: "K1F pairs"}.get(depth, "single steps"),
                             single_vecs, gram_vecs, upd_vecs),
            "mix": "%d reads : %d writes per launch" % mixrw,
            "mix_ceiling_gbs": mc[0], "mix_ceiling_source": mc[1],
            "frac_of_mix_ceiling": (k1["achieved_gbs"] / mc[0]) if (mc[0] and k1["achieved_gbs"]) else None,
            "path_bytes_per_step": path_bytes,
            "path_achieved_gbs": path_bytes / (st.ms_total / a.steps / 1e3) / 1e9,
            "path_frac": path_bytes / (st.ms_total / a.steps / 1e3) / 1e9 / peak}
    # SURVEY 8(d)'s byte contract as written (single steps with stored W: 4 vectors per basis step,
    # 3 at j = 0 and 2 at j = s-1; Gram 2s; update 2s+3; 8s per outer, + s face sets for varcoef7)
    # beside the schedule's own bytes above: the schedule moves fewer vectors
    # (W-free Gram, recurrence update, K1M triples), so against 8(d) a fraction above 1 is expected
    t_outer = st.ms_total / a.steps / 1e3
    c8_basis = (4 * s - 3) * vec + s * face_bytes
    c8 = {"basis": c8_basis, "gram": 2 * s * vec, "update": (2 * s + 3) * vec}
    # 8(d)'s per-launch K1 bytes for the dominant kernel: 4 vectors per basis step it runs
    c8_k1 = 4 * depth * vec
    roof["contracts"] = {
        "schedule": {"vectors_per_outer": {"basis": basis_vecs, "gram": gram_vecs, "update": upd_vecs},
                     "bytes_per_outer": path_bytes, "achieved_gbs": path_bytes / t_outer / 1e9,
                     "frac": path_bytes / t_outer / 1e9 / peak,
                     "dominant_kernel_frac": k1["frac"]},
        "survey_8d": {"vectors_per_outer": {"basis": 4 * s - 3, "gram": 2 * s, "update": 2 * s + 3},
                      "bytes_per_outer": sum(c8.values()), "achieved_gbs": sum(c8.values()) / t_outer / 1e9,
                      "frac": sum(c8.values()) / t_outer / 1e9 / peak,
                      "dominant_kernel_frac": c8_k1 / (k1["ms_per_launch"] / 1e3) / 1e9 / peak
                                              if k1["ms_per_launch"] else None,
                      "note": "SURVEY 8(d) counts as written (stored W, single basis steps); the kernels move the "
                              "schedule's vectors, so this 'fraction' is not a physical bandwidth (> 1 possible)"}}
    if a.kind == "5pt":
        roof["us_per_outer"] = 1e3 * st.ms_total / a.steps
        roof["note"] = "cfg 1: the working set lives in L2; the metric is latency per outer iteration (SURVEY 8(d))"
    # end-to-end: host b in, host x out, through the C ABI (sscg_solve_host)
    e2e = None
    if not a.no_e2e:
        xh = torch.empty(n_local, dtype=torch.float64).pin_memory()
        bh = b_host.numpy()
        S.solve_host(bh, xh.numpy(), rtol=0.0, max_outer=1)   # untimed: the call's staging buffers are allocated once
        barrier()
        t0 = time.perf_counter()
        S.solve_host(bh, xh.numpy(), rtol=0.0, max_outer=a.steps)
        t1 = time.perf_counter()
        te = max_over_ranks(dist, t1 - t0)
        e2e = {"value": n_global * a.steps / te / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": 8.0 * n_local / a.steps, "d2h_bytes_per_step": 8.0 * n_local / a.steps,
               "note": f"one sscg_solve_host call: b H2D, {a.steps} outer iterations (+ final stopping-test "
                       "basis/Gram), x D2H; host wall clock, max over ranks"}
    S.close()
    if dist:
        dist.barrier()
    if rank != 0:
        if dist:
            dist.destroy_process_group()
        return
    cpu = None
    if world == 1 and not a.no_cpu_baseline:
        hi = host_info()
        # the oracle at the full one-GPU size, 3 outer iterations,
        # when the host has the memory (the oracle holds P and W: 2s+4 vectors);
        # else ~10 s of CPU work on 64 planes of the same n x n grid
        need_gb = (2 * s + 6) * 8.0 * n * n * (1 if a.kind == "5pt" else n) / 1e9
        if a.kind == "5pt":
            v, per, desc = oracle_sample(a, 200, 5)
        elif hi.get("MemAvailable_GB", 0.0) >= 1.6 * need_gb and not a.strong:
            v, per, desc = oracle_sample(a, 3, 0, planes=n)
        else:
            v, per, desc = oracle_sample(a, 24, 1, planes=64)
        cpu = {"value": v, "unit": UNIT, "cores": cpu_cores(), "kind": "oracle", "sample": desc, "cpu": cpu_model(),
               "ms_per_outer": per * 1e3, "host": hi}
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic", "config": cfg, "roofline": roof,
            "kernels": kern, "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": launches,
            "clocks": clk.summary(), "impl": "ours",
            # the s-independent rate for constant-coefficient stencils
            "gdof_step_per_s": value * s}
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
