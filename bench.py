#!/usr/bin/env python3
"""bench.py -- encrypted 64x64x64 HEGMM products per second (BFV N=8192) on B200.

Workload (BASELINE.json configs[3], "cfg4"): a batch of 4096 independent
A(64x64).B(64x64) products, entries uniform in [-8, 7] drawn per instance with
the reference campaign's splitmix64 streams (paper_2405_02238_b200/workload.py),
BFV N=8192, t=65537, Q = 3 x 60-bit primes (+1 special prime, dnum 3), keys
replicated on every GPU, instances sharded across ranks (strong scaling: the
4096 are split N ways), result ciphertexts gathered to rank 0 over NCCL.
A "step" is the cloud phase of HEGMM (basic_mm, Algorithm 1:
proj/src/algorithms.cpp:233-242 -- every rotation, mask product, CC-mult and
accumulation) over the whole batch, its encrypted inputs resident in HBM.

  value : step throughput, CUDA-event time on the library stream, max over ranks
  e2e   : the same products through the C ABI with HOST buffers
          (hgm_matmul_batch: host A, B -> pack -> H2D -> encrypt -> cloud ->
          decrypt -> D2H -> host C), wall time between barriers, max over ranks
  roofline : the NTT kernel (dominant kernel class) vs measured HBM bandwidth
  cpu_baseline : the reference's own basic_mm (compiled from its sources,
          oracle/_ref) over the CPU BFV restatement, one bounded sample on 1 core

--impl reference runs that CPU path on all host threads (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "encrypted 64x64x64 matmuls/sec (BFV N=8192)"
UNIT = "matmuls/s"
M = L_ = N_ = 64
LO, HI = -8, 7
TOTAL_INSTANCES = 4096
SEED = 20240404
PARAM_ID = 0  # N 8192 / Q 3x60-bit / P 1x60-bit / dnum 3
LIMB_BYTES = 2 * 8 * 8192  # algorithmic bytes of one N=8192 limb NTT (read + write)
OP_BYTES_PER_MATMUL = 1.2445e9  # SURVEY.md 8(d), cfg2/cfg4 basic_mm


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def sm_max_mhz(device: int = 0) -> float:
    """The GPU's maximum SM clock (nvidia-smi clocks.max.sm); 1965 MHz (B200) if unreadable."""
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.max.sm", "--format=csv,noheader,nounits", "-i",
                              str(device)], capture_output=True, text=True, timeout=5).stdout
        return float(out.strip().splitlines()[0])
    except Exception:
        return 1965.0


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled DURING the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                      "-i", str(self.device)], capture_output=True, text=True, timeout=5).stdout
                parts = [p.strip() for p in out.strip().split(",")]
                if len(parts) == 6:
                    self.samples.append(parts)
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


from paper_2405_02238_b200.dist import comm_from_env, counter_base, env_rank, shard  # noqa: E402


def cpu_baseline(seconds_budget: float = 20.0):
    """The reference's basic_mm over the CPU BFV restatement: 1 core, bounded sample."""
    from oracle.bindings import OracleSession, RefLib  # CPU baseline leg only
    from paper_2405_02238_b200.workload import batch

    if not RefLib.available():
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "port",
                "sample": "unavailable: oracle/_ref not built"}
    sess = OracleSession(PARAM_ID, 1)
    A, B = batch(SEED, 0, 8, M, L_, N_, LO, HI)
    sess.mm(A[0], B[0], "basic", counter0=0)  # keys, tables (not timed)
    done, t0 = 0, time.perf_counter()
    while done < len(A) and (done == 0 or time.perf_counter() - t0 < seconds_budget):
        C = sess.mm(A[done], B[done], "basic", counter0=3 * done)
        assert np.array_equal(C, (A[done] @ B[done]) % 65537)
        done += 1
    dt = time.perf_counter() - t0
    sess.close()
    return {"value": done / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{done} x cfg4 instance(s) through the reference basic_mm (compiled from "
                      f"/root/reference sources) over the CPU RNS-BFV restatement (oracle/), "
                      f"1 thread, {dt:.1f} s",
            "cleartext_emulator": cleartext_emulator_rate()}


def cleartext_emulator_rate(seconds_budget: float = 3.0):
    """BASELINE.md's literal reference CPU path: the reference's own basic_mm on
    its cleartext slot emulator (SlotBackend{4096, 65537}), 1 thread.  Not an
    encrypted product -- reported for context only."""
    from oracle.bindings import RefLib  # CPU baseline leg only
    from paper_2405_02238_b200.workload import batch

    A, B = batch(SEED, 0, 64, M, L_, N_, LO, HI)
    RefLib.mm(A[0], B[0], "basic", slots=4096)
    done, t0 = 0, time.perf_counter()
    while done < len(A) and (done == 0 or time.perf_counter() - t0 < seconds_budget):
        C, _ = RefLib.mm(A[done], B[done], "basic", slots=4096)
        assert np.array_equal(C, (A[done] @ B[done]) % 65537)
        done += 1
    dt = time.perf_counter() - t0
    return {"value": done / dt, "unit": UNIT, "cores": 1,
            "sample": f"{done} x cfg4 instance(s), reference basic_mm on SlotBackend{{4096, 65537}} "
                      f"(cleartext slot emulator, NOT homomorphic), 1 thread, {dt:.1f} s"}


def run_reference(args):
    """--impl reference: the reference CPU path on all host threads (rank 0 only)."""
    rank = env_int("RANK", 0)
    if rank != 0:
        return 0
    from oracle.bindings import OracleSession, RefLib
    from paper_2405_02238_b200.workload import batch

    if not RefLib.available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libhegmm_ref.so was not built"}))
        return 0
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    threads = max(1, cores)
    sessions = [None] * threads

    def init(i):
        sessions[i] = OracleSession(PARAM_ID, 1)
        A, B = batch(SEED, i, 1, M, L_, N_, LO, HI)
        sessions[i].mm(A[0], B[0], "basic", counter0=0)  # keygen warm-up

    ts = [threading.Thread(target=init, args=(i,)) for i in range(threads)]
    [t.start() for t in ts]
    [t.join() for t in ts]
    # one step = one product per thread (a bounded sample of the 4096-instance workload)
    step_times = []
    nxt = [0]
    for step in range(args.warmup + args.steps):
        A, B = batch(SEED, step * threads, threads, M, L_, N_, LO, HI)
        errs = []

        def work(i):
            C = sessions[i].mm(A[i], B[i], "basic", counter0=3 * (step * threads + i))
            if not np.array_equal(C, (A[i] @ B[i]) % 65537):
                errs.append(i)

        t0 = time.perf_counter()
        ws = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        [w.start() for w in ws]
        [w.join() for w in ws]
        dt = time.perf_counter() - t0
        if errs:
            raise RuntimeError(f"reference path produced wrong products for {errs}")
        if step >= args.warmup:
            step_times.append(dt)
        nxt[0] += threads
    total = sum(step_times)
    value = threads * len(step_times) / total
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / len(step_times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64",
        "data": "synthetic (reference campaign splitmix64 draws)",
        "config": {"workload": "cfg4: 64x64x64 HEGMM (basic_mm) instances, BFV N=8192 t=65537 3x60b",
                   "per_step": f"{threads} instances (1 per host thread)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{threads} threads x 1 instance per step: the reference basic_mm "
                                   f"(compiled from /root/reference sources) over the CPU RNS-BFV "
                                   f"restatement (oracle/)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    for s in sessions:
        s.close()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="cfg4", choices=["cfg4", "cfg5"])
    ap.add_argument("--algo", default=None, choices=["basic", "enhanced"])
    ap.add_argument("--instances", type=int, default=None,
                    help="products per GPU per step (cfg4: 4096 instances; cfg5: 128^3 products)")
    ap.add_argument("--strong", action="store_true",
                    help="split --instances across the GPUs instead of giving every GPU that many")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rules: >= 3 warm-up steps
    if args.impl == "reference":
        return run_reference(args)
    if args.config == "cfg5":
        return run_cfg5(args)
    return run_cfg4(args)


def ntt_roofline(ctx, limb_bytes, label):
    """Forward / inverse NTT and the key-switch inner product timed live (CUDA
    events on the library stream), inputs larger than L2 with canonical random
    residues; algorithmic bytes per unit from SURVEY.md 8(d) / DESIGN.md."""
    peak, peak_src = load_peaks()
    limbs = 148 * 8 * 4  # 4736 limbs: > 126 MB L2 at N = 8192, several waves of 444 resident CTAs
    if ctx.N > 8192:
        limbs = 148 * 8
    ntt_ms = ctx.bench_ntt(limbs, 20, True)
    intt_ms = ctx.bench_ntt(limbs, 20, False)
    achieved = limbs * limb_bytes / (ntt_ms / 1e3) / 1e9
    # key switch, compulsory bytes per rotation: read dnum (L+K) digit limbs + L c0 limbs, write
    # 2 (L+K) accumulator limbs, and the dnum 2 (L+K)-limb Galois key once per group of 8
    # rotations that share it (the kernel's key reuse; DESIGN.md roofline table)
    R = ctx.L + ctx.K
    ks_items = 2048 if ctx.N == 8192 else 256
    ks_bytes = (ctx.dnum * R + ctx.L + 2 * R + ctx.dnum * 2 * R / 8) * ctx.N * 8
    ks_ms = ctx.bench_keyswitch(ks_items, 10)
    ks_gbs = ks_items * ks_bytes / (ks_ms / 1e3) / 1e9
    # the in-step key-switch kernel: masked sums of rotations straight from the ModUp digits
    # (k_ks_plan), as the cloud step lays them out -- tiles of 16 instances, every sum of an
    # instance reading that instance's digits, masked keys read once per tile.  Compulsory
    # bytes per sum: 2 (L+K) limbs written, terms (2 dnum (L+K) + L) masked-key limbs per
    # tile, the instance's dnum (L+K) + L digit / c0 limbs once per `sums` sums.
    pl_inst, pl_sums, pl_terms, pl_tile = (128, 63, 2, 16) if ctx.N == 8192 else (16, 16, 2, 16)
    pl_bytes = (2 * R + pl_terms * (2 * ctx.dnum * R + ctx.L) / pl_tile
                + (ctx.dnum * R + ctx.L) / pl_sums) * ctx.N * 8
    pl_ms = ctx.bench_keyswitch_plan(pl_inst, pl_sums, pl_terms, pl_tile, 5)
    pl_n = pl_inst * pl_sums
    pl_gbs = pl_n * pl_bytes / (pl_ms / 1e3) / 1e9
    # what the same sums cost as separate kernels (one k_ks_inner per rotation, then the
    # masked sum of the accumulators): the bytes k_ks_plan no longer moves
    unfused = pl_terms * ks_bytes + (pl_terms * (2 * R + R) + 2 * R) * ctx.N * 8
    # integer-multiply ceiling of the butterfly: 22 fmaheavy cycles per warp-butterfly
    # (3 IMAD.WIDE + IMAD.HI at 4, 3 IMAD at 2), 4 SMSPs x 148 SMs
    logn = ctx.N.bit_length() - 1
    SM_MAX_MHZ = sm_max_mhz()
    warp_bf = limbs * (ctx.N // 2) * logn / 32
    traffic, pipes = None, None
    prof = os.path.join(ROOT, "profiles", "ntt_traffic.json")
    if os.path.exists(prof):
        try:
            rec = json.load(open(prof))
            if rec.get("N", 8192) == ctx.N and rec.get("bytes_per_limb"):
                traffic = rec["bytes_per_limb"] * limbs
                # integer-pipe utilisation of the same launch (ncu, profiles/): the bound that binds
                pipes = {k: rec.get(k) for k in ("fmaheavy_frac", "alu_frac", "issue_frac")}
                pipes["source"] = rec.get("source")
        except Exception:
            traffic = None
    return {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic,
            "kernel": label, "algorithmic_bytes_per_launch": limbs * limb_bytes, "limbs_per_launch": limbs,
            "ms_per_launch": round(ntt_ms, 4),
            "inverse_frac": round(limbs * limb_bytes / (intt_ms / 1e3) / 1e9 / peak, 4),
            "peak_source": peak_src, "frac_vs_spec_8tbs": round(achieved / 8000.0, 4),
            "int_pipes_ncu": pipes,
            "int_multiply_ceiling": {"pipe": "fmaheavy (IMAD / IMAD.WIDE / IMAD.HI)",
                                     "cycles_per_warp_butterfly": 22,
                                     "min_ms_at_max_clock": round(warp_bf * 22 / (148 * 4) / (SM_MAX_MHZ * 1e3), 4),
                                     "frac_of_ceiling": round(warp_bf * 22 / (148 * 4) / (SM_MAX_MHZ * 1e3) / ntt_ms, 4),
                                     "ceiling_as_hbm_frac": round(limbs * limb_bytes / (warp_bf * 22 / (148 * 4) / (SM_MAX_MHZ * 1e6)) / 1e9 / peak, 4)},
            "keyswitch_plan": {"kernel": "k_ks_plan (masked sum of rotations as one key inner product over masked "
                                         "keys; the cloud step's key-switch kernel for cached programs)",
                               "sums_per_launch": pl_n, "terms_per_sum": pl_terms, "tile": pl_tile,
                               "algorithmic_bytes_per_sum": int(pl_bytes), "ms_per_launch": round(pl_ms, 4),
                               "achieved": round(pl_gbs, 1), "frac": round(pl_gbs / peak, 4),
                               "unfused_bytes_per_sum": int(unfused),
                               "unfused_equivalent_gbs": round(pl_n * unfused / (pl_ms / 1e3) / 1e9, 1),
                               "traffic": plan_traffic(ctx.N, pl_n), "int_pipes_ncu": plan_pipes(ctx.N)},
            "keyswitch": {"kernel": "k_ks_inner (key inner product of one rotation, Galois gather fused, 8 rotations per key read; relinearisation and uncached programs)",
                          "rotations_per_launch": ks_items, "algorithmic_bytes_per_rotation": int(ks_bytes),
                          "traffic": ks_traffic(ctx.N, ks_items), "int_pipes_ncu": ks_pipes(ctx.N),
                          "ms_per_launch": round(ks_ms, 4), "achieved": round(ks_gbs, 1),
                          "frac": round(ks_gbs / peak, 4)}}


def ks_traffic(N, items):
    """DRAM bytes per k_ks_inner launch from the committed ncu --set full capture
    (profiles/ks_traffic.json), scaled to `items` rotations; None if absent."""
    prof = os.path.join(ROOT, "profiles", "ks_traffic.json")
    try:
        rec = json.load(open(prof))
        if rec.get("N") == N and rec.get("bytes_per_rotation"):
            return rec["bytes_per_rotation"] * items
    except Exception:
        pass
    return None


def plan_traffic(N, sums):
    """DRAM bytes per k_ks_plan launch from the committed ncu --set full capture of the
    same launch (profiles/ks_plan_traffic.json); None if absent."""
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "ks_plan_traffic.json")))
        if rec.get("N") == N and rec.get("bytes_per_sum"):
            return rec["bytes_per_sum"] * sums
    except Exception:
        pass
    return None


def plan_pipes(N):
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "ks_plan_traffic.json")))
        if rec.get("N") == N:
            return {k: rec.get(k) for k in ("fmaheavy_frac", "alu_frac", "issue_frac", "dram_frac", "source")}
    except Exception:
        pass
    return None


def ks_pipes(N):
    try:
        rec = json.load(open(os.path.join(ROOT, "profiles", "ks_traffic.json")))
        if rec.get("N") == N:
            return {k: rec.get(k) for k in ("fmaheavy_frac", "alu_frac", "issue_frac")}
    except Exception:
        pass
    return None


def run_cfg4(args):
    import paper_2405_02238_b200 as hb
    from paper_2405_02238_b200.workload import batch

    rank, world, local = env_rank()
    algo_name = args.algo or "basic"
    algo = hb.ALGOS[algo_name]
    per_gpu = args.instances or TOTAL_INSTANCES
    total = per_gpu if args.strong else per_gpu * world
    first, count = shard(rank, world, total)
    local = env_int("HGM_DEVICE", local)  # test hook: several ranks on one GPU (tests/test_gpu_multirank.py)
    ctx = hb.Context(PARAM_ID, 1, local)
    comm = comm_from_env(ctx)  # the library's NCCL communicator (no torch)
    A, B = batch(SEED, first, count, M, L_, N_, LO, HI)
    st, facts = hb.program_info(algo, M, L_, N_, ctx.slot_count, ctx.N)
    E = facts["encryptions"]

    def barrier():
        ctx.sync()
        if comm:
            comm.barrier()

    def max_over_ranks(x: float) -> float:
        return comm.max(x) if comm else x

    # ---------------------------------------------------------------- value: cloud phase
    bt = hb.Batch(ctx, A, B, algo=algo, counter0=counter_base(first, E))  # client phase (not timed)
    for _ in range(args.warmup):
        bt.cloud()
    barrier()
    launches0 = ctx.launch_count()
    step_ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            step_ms.append(bt.cloud())
    launches = ctx.launch_count() - launches0
    barrier()
    total_ms = max_over_ranks(sum(step_ms))
    value = total * args.steps / (total_ms / 1e3)
    # correctness of what was timed (decrypt outside the timed region): every product
    want = np.einsum("kij,kjl->kil", A, B) % 65537
    C = bt.decrypt()
    wrong = int(np.count_nonzero(~np.all(C == want, axis=(1, 2))))
    if wrong:
        raise RuntimeError(f"timed cloud phase produced {wrong} wrong products")
    verified = {"value": f"{count} of {count} products decrypted and checked (rank {rank})"}
    # gather every rank's result ciphertexts to rank 0 over the library's NCCL
    # communicator (the only collective); rank 0 decrypts all of them
    gather_ms = None
    if comm:
        barrier()
        t0 = time.perf_counter()
        ptr, n = comm.gather_batch(bt, root=0)
        gather_ms = 1e3 * (time.perf_counter() - t0)
        gather_ms = max_over_ranks(gather_ms)
        if rank == 0:
            try:
                Cg = ctx.decrypt_products(ptr, n, M, L_, N_, algo=algo)
            finally:
                comm.free_buffer(ptr)
            Ag, Bg = batch(SEED, 0, total, M, L_, N_, LO, HI)
            wantg = np.einsum("kij,kjl->kil", Ag, Bg) % 65537
            wrong = int(np.count_nonzero(~np.all(Cg == wantg, axis=(1, 2))))
            if n != total or wrong:
                raise RuntimeError(f"gathered {n} of {total} ciphertexts, {wrong} decrypt wrongly")
            verified["gather"] = f"{n} of {total} ciphertexts gathered to rank 0 over NCCL, all decrypted and checked"
    bt.free()

    # ---------------------------------------------------------------- e2e through the C ABI
    e2e = None
    if not args.no_e2e:
        # warm-up at the full size like the timed steps: the first full call grows the
        # stream-ordered memory pool and the pinned staging to this path's chunk size
        for _ in range(args.warmup):
            ctx.matmul_batch(A, B, algo=algo, counter0=first * E)
        e2e_times = []
        for s in range(args.steps):
            barrier()
            t0 = time.perf_counter()
            Ce, _ = ctx.matmul_batch(A, B, algo=algo, counter0=first * E)
            e2e_times.append(time.perf_counter() - t0)
        barrier()
        e2e_total = max_over_ranks(sum(e2e_times))
        wrong = int(np.count_nonzero(~np.all(Ce == want, axis=(1, 2))))  # outside the timed region
        if wrong:
            raise RuntimeError(f"e2e path produced {wrong} wrong products")
        verified["e2e"] = f"{count} of {count} products of the last step checked (rank {rank})"
        # bytes the library moves: slot vectors go up as u32 residues mod t (N/2 per
        # encryption, pinned staging) and decrypted rows come back as N/2 u32 each
        h2d = total * E * ctx.slot_count * 4
        d2h = total * ctx.slot_count * 4
        e2e = {"value": total * args.steps / e2e_total, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "hgm_matmul_batch (C ABI): host int64 A,B -> host C, incl. client encrypt/decrypt"}

    roofline = ntt_roofline(ctx, LIMB_BYTES, "k_ntt_fwd3<13> (forward NTT, N=8192, 64-bit Shoup, 3 CTAs/SM)")
    roofline["op_level"] = {"bytes_per_matmul": OP_BYTES_PER_MATMUL,
                            "achieved": round(value * OP_BYTES_PER_MATMUL / 1e9 / world, 1),
                            "unit": "GB/s per GPU",
                            "frac": round(value * OP_BYTES_PER_MATMUL / 1e9 / world / roofline["peak"], 4)}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong" if args.strong else "weak", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (reference campaign splitmix64 draws, seed %d)" % SEED,
            "config": {"workload": f"cfg4: {per_gpu} x A(64x64).B(64x64) {algo_name}_mm instances "
                                   f"{'in total' if args.strong else 'per GPU'}, BFV N=8192 t=65537 "
                                   f"Q=3x60b P=1x60b dnum=3 (log2 PQ ~ 240: above the 128-bit bound for N=8192, "
                                   f"as BASELINE.json's 3x60-bit Q prescribes)",
                       "instances_per_step": total, "instances_per_gpu": count, "algo": algo_name,
                       "cloud_ops_per_instance": {"rot": int(st[7]), "cmult": int(st[5]), "add": int(st[1]),
                                                  "mult": int(st[3])},
                       "rotations_after_cse": facts["rotations"], "parallelism": f"instances x{world}",
                       "l2": "inputs larger than L2 (%.1f GB of ciphertexts per GPU per step)" %
                             (count * E * ctx.ct_words * 8 / 1e9)},
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk.summary(),
            "roofline": roofline,
            "cpu_baseline": None if args.no_cpu_baseline or world > 1 else cpu_baseline(),
        }
        line["verified"] = verified
        if gather_ms is not None:
            line["nccl_gather_ms"] = round(gather_ms, 3)
        print(json.dumps(line))
    if comm:
        comm.barrier()
        comm.close()
    ctx.close()
    return 0


CFG5 = dict(m=128, l=128, n=128, lo=-4, hi=3, param_id=1, parts=8, seed=20240505)


def run_cfg5(args):
    """Config 5: A(128x128).B(128x128) at N=32768 (8 x ~55-bit Q, 4 special
    primes, dnum 2), HEGMM-Enhanced over 8 row blocks of 16 rows:
    a step runs `--instances` such products (default 4) -- 8 row-block
    products each, sharded over the ranks -- and gathers the result ciphertexts
    to rank 0 over the library's NCCL communicator."""
    import paper_2405_02238_b200 as hb
    from paper_2405_02238_b200.dist import row_blocks
    from paper_2405_02238_b200.workload import splitmix_matrices

    rank, world, local = env_rank()
    c = CFG5
    algo_name = args.algo or "enhanced"
    algo = hb.ALGOS[algo_name]
    products = args.instances or 4
    total_blocks = products * c["parts"]
    first, count = shard(rank, world, total_blocks)
    h = c["m"] // c["parts"]
    local = env_int("HGM_DEVICE", local)
    ctx = hb.Context(c["param_id"], 1, local)
    comm = comm_from_env(ctx)
    mats = [splitmix_matrices(c["seed"], p, c["m"], c["l"], c["n"], c["lo"], c["hi"]) for p in range(products)]
    blocks = row_blocks(c["m"], c["parts"])
    As = np.stack([mats[b // c["parts"]][0][blocks[b % c["parts"]][0]: blocks[b % c["parts"]][0] + h]
                   for b in range(first, first + count)])
    Bs = np.stack([mats[b // c["parts"]][1] for b in range(first, first + count)])
    st, facts = hb.program_info(algo, h, c["l"], c["n"], ctx.slot_count, ctx.N)
    E = facts["encryptions"]

    def barrier():
        ctx.sync()
        if comm:
            comm.barrier()

    bt = hb.Batch(ctx, As, Bs, algo=algo, counter0=first * E)
    for _ in range(args.warmup):
        bt.cloud()
    barrier()
    launches0 = ctx.launch_count()
    step_ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            step_ms.append(bt.cloud())
    launches = ctx.launch_count() - launches0
    barrier()
    total_ms = comm.max(sum(step_ms)) if comm else sum(step_ms)
    value = products * args.steps / (total_ms / 1e3)
    # gather to rank 0, decrypt, stitch and check every product (outside the timed region)
    verified = {}
    if comm:
        ptr, n = comm.gather_batch(bt, root=0)
        if rank == 0:
            try:
                Cb = ctx.decrypt_products(ptr, n, h, c["l"], c["n"], algo=algo)
            finally:
                comm.free_buffer(ptr)
    else:
        Cb = bt.decrypt()
    if rank == 0:
        for p in range(products):
            Cp = np.concatenate(list(Cb[p * c["parts"]:(p + 1) * c["parts"]]))
            if not np.array_equal(Cp, (mats[p][0] @ mats[p][1]) % 65537):
                raise RuntimeError(f"cfg5 product {p} decrypts wrongly")
        verified["value"] = f"{products} of {products} 128^3 products (gathered to rank 0) decrypted and checked"
    bt.free()
    e2e = None
    if not args.no_e2e:
        for _ in range(args.warmup):  # full-size warm-up, as for the timed steps
            ctx.matmul_batch(As, Bs, algo=algo, counter0=first * E)
        times = []
        for _ in range(args.steps):
            barrier()
            t0 = time.perf_counter()
            Ce, _ = ctx.matmul_batch(As, Bs, algo=algo, counter0=first * E)
            times.append(time.perf_counter() - t0)
        barrier()
        tot = comm.max(sum(times)) if comm else sum(times)
        want = np.einsum("kij,kjl->kil", As, Bs) % 65537
        if not np.array_equal(Ce, want):
            raise RuntimeError("cfg5 e2e path produced wrong row blocks")
        verified["e2e"] = f"{count} of {count} row blocks of the last step checked (rank {rank})"
        e2e = {"value": products * args.steps / tot, "unit": "matmuls/s",
               "h2d_bytes_per_step": total_blocks * E * ctx.slot_count * 4,
               "d2h_bytes_per_step": total_blocks * ctx.slot_count * 4,
               "path": "hgm_matmul_batch (C ABI) over the rank's row blocks: host int64 in -> host C"}
    roofline = ntt_roofline(ctx, 2 * 8 * ctx.N,
                            "k_ntt_fwd_c4<13> (forward NTT, N=32768, one HBM pass: 4-CTA clusters, outer stages through DSMEM, 64-bit Shoup)")
    if rank == 0:
        line = {
            "metric": "encrypted 128x128x128 matmuls/sec (BFV N=32768)", "value": round(value, 3),
            "unit": "matmuls/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (reference campaign splitmix64 draws, seed %d)" % c["seed"],
            "config": {"workload": f"cfg5: {products} x A(128x128).B(128x128) {algo_name}_mm per step as "
                                   f"{total_blocks} row-block products 16x128.128x128, BFV N=32768 t=65537 "
                                   f"Q=8x55b P=4x55b dnum=2", "row_blocks_per_gpu": count,
                       "cloud_ops_per_row_block": {"rot": int(st[7]), "cmult": int(st[5]), "add": int(st[1]),
                                                   "mult": int(st[3])},
                       "parallelism": f"row blocks x{world}",
                       "l2": "inputs larger than L2 (%.2f GB of ciphertexts per GPU)" %
                             (count * E * ctx.ct_words * 8 / 1e9)},
            "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(), "roofline": roofline,
            "cpu_baseline": None, "verified": verified,
        }
        print(json.dumps(line))
    if comm:
        comm.barrier()
        comm.close()
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
