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


from paper_2405_02238_b200.dist import counter_base, gather_ciphertexts, shard  # noqa: E402


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
                      f"1 thread, {dt:.1f} s"}


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
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u64",
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
    ap.add_argument("--algo", default="basic", choices=["basic", "enhanced"])
    ap.add_argument("--instances", type=int, default=TOTAL_INSTANCES)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rules: >= 3 warm-up steps
    if args.impl == "reference":
        return run_reference(args)

    import paper_2405_02238_b200 as hb
    from paper_2405_02238_b200.workload import batch

    rank, world, local = env_int("RANK", 0), env_int("WORLD_SIZE", 1), env_int("LOCAL_RANK", 0)
    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist

        torch.cuda.set_device(local)
        tdist.init_process_group("nccl", device_id=torch.device("cuda", local))
        dist = tdist

    algo = hb.ALGOS[args.algo]
    first, count = shard(rank, world, args.instances)
    ctx = hb.Context(PARAM_ID, 1, local)
    A, B = batch(SEED, first, count, M, L_, N_, LO, HI)
    st, facts = hb.program_info(algo, M, L_, N_, ctx.slot_count, ctx.N)
    E = facts["encryptions"]

    def barrier():
        if dist:
            import torch

            torch.cuda.synchronize()
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not dist:
            return x
        import torch

        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---------------------------------------------------------------- value: cloud phase
    bt = hb.Batch(ctx, A, B, algo=algo, counter0=counter_base(first, E))  # client phase (not timed)
    for _ in range(args.warmup):
        bt.cloud()
    barrier()
    ctx.sync()
    launches0 = ctx.launch_count()
    step_ms = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            step_ms.append(bt.cloud())
    launches = ctx.launch_count() - launches0
    ctx.sync()
    barrier()
    total_ms = max_over_ranks(sum(step_ms))
    value = args.instances * args.steps / (total_ms / 1e3)
    # correctness of what was timed (decrypt outside the timed region): every product
    want = np.einsum("kij,kjl->kil", A, B) % 65537
    C = bt.decrypt()
    wrong = int(np.count_nonzero(~np.all(C == want, axis=(1, 2))))
    if wrong:
        raise RuntimeError(f"timed cloud phase produced {wrong} wrong products")
    verified = {"value": f"{count} of {count} products decrypted and checked"}
    # gather result ciphertexts to rank 0 over NCCL (the only collective)
    gather_ms = None
    if dist:
        import torch

        W = ctx.ct_words

        class _View:
            def __init__(self, ptr, n):
                self.__cuda_array_interface__ = {"shape": (n,), "typestr": "<i8", "data": (ptr, False),
                                                 "version": 3}

        mine = torch.as_tensor(_View(bt.output_ptr(0), count * W), device="cuda")
        ctx.sync()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        got = gather_ciphertexts(dist, mine, count, W, args.instances, world, rank, device="cuda")
        torch.cuda.synchronize()
        gather_ms = 1e3 * (time.perf_counter() - t0)
        if rank == 0:  # rank 0 (the client side) decrypts a sample of every shard
            for r, part in enumerate(got):
                f, c = shard(r, world, args.instances)
                if c:  # check the shard's first product from its gathered ciphertext
                    slots = ctx.decrypt_words(part[: W], facts["segment"])[0]
                    Ar, Br = batch(SEED, f, 1, M, L_, N_, LO, HI)
                    col = facts["order"] == 0
                    C0 = np.array([[slots[(i + j * M) if col else (i * N_ + j)] for j in range(N_)]
                                   for i in range(M)])
                    if not np.array_equal(C0, (Ar[0] @ Br[0]) % 65537):
                        raise RuntimeError(f"gathered ciphertext of rank {r} decrypts wrongly")
    bt.free()

    # ---------------------------------------------------------------- e2e through the C ABI
    e2e = None
    if not args.no_e2e:
        ctx.matmul_batch(A[:8], B[:8], algo=algo)  # warm program/mask caches
        e2e_times = []
        for s in range(args.steps):
            barrier()
            t0 = time.perf_counter()
            Ce, _ = ctx.matmul_batch(A, B, algo=algo, counter0=first * E)
            barrier()
            e2e_times.append(time.perf_counter() - t0)
        e2e_total = max_over_ranks(sum(e2e_times))
        wrong = int(np.count_nonzero(~np.all(Ce == want, axis=(1, 2))))  # outside the timed region
        if wrong:
            raise RuntimeError(f"e2e path produced {wrong} wrong products")
        verified["e2e"] = f"{count} of {count} products of the last step checked"
        # bytes the library moves: slot vectors go up as u32 residues mod t (N/2 per
        # encryption, pinned staging) and decrypted rows come back as N/2 u32 each
        h2d = args.instances * E * ctx.slot_count * 4
        d2h = args.instances * ctx.slot_count * 4
        e2e = {"value": args.instances * args.steps / e2e_total, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "path": "hgm_matmul_batch (C ABI): host int64 A,B -> host C, incl. client encrypt/decrypt"}

    # ---------------------------------------------------------------- roofline: NTT kernel
    limbs = 148 * 8
    ntt_ms = ctx.bench_ntt(limbs, 20, True)
    intt_ms = ctx.bench_ntt(limbs, 20, False)
    peak, peak_src = load_peaks()
    achieved = limbs * LIMB_BYTES / (ntt_ms / 1e3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ntt_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get("bytes_per_limb")
            traffic = traffic * limbs if traffic else None
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": "k_ntt_fwd3<13> (forward NTT, N=8192, 64-bit Shoup, 3 CTAs/SM)",
                "algorithmic_bytes_per_launch": limbs * LIMB_BYTES, "limbs_per_launch": limbs,
                "inverse_frac": round(limbs * LIMB_BYTES / (intt_ms / 1e3) / 1e9 / peak, 4),
                "peak_source": peak_src,
                "frac_vs_spec_8tbs": round(achieved / 8000.0, 4),
                # op-level bytes of one cfg2/cfg4 basic_mm matmul
                # (every primitive's compulsory ciphertext/key/mask traffic x the reference op
                # counts); fused, deduplicated execution may move fewer, so frac may exceed 1
                "op_level": {"bytes_per_matmul": OP_BYTES_PER_MATMUL,
                             "achieved": round(value * OP_BYTES_PER_MATMUL / 1e9 / world, 1),
                             "unit": "GB/s per GPU",
                             "frac": round(value * OP_BYTES_PER_MATMUL / 1e9 / world / peak, 4)}}

    if rank == 0:
        clocks = clk.summary()
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(total_ms / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u64",
            "data": "synthetic (reference campaign splitmix64 draws, seed %d)" % SEED,
            "config": {"workload": f"cfg4: {args.instances} x A(64x64).B(64x64) {args.algo}_mm instances, "
                                   f"BFV N=8192 t=65537 Q=3x60b P=1x60b dnum=3",
                       "instances_per_step": args.instances, "algo": args.algo,
                       "cloud_ops_per_instance": {"rot": int(st[7]), "cmult": int(st[5]), "add": int(st[1]),
                                                  "mult": int(st[3])},
                       "rotations_after_cse": facts["rotations"], "parallelism": f"instances x{world}",
                       "l2": "inputs larger than L2 (%.1f GB of ciphertexts per step)" %
                             (args.instances * E * ctx.ct_words * 8 / 1e9)},
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "roofline": roofline,
            "cpu_baseline": None if args.no_cpu_baseline or world > 1 else cpu_baseline(),
        }
        line["verified"] = verified
        if gather_ms is not None:
            line["nccl_gather_ms"] = round(gather_ms, 3)
        print(json.dumps(line))
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()
    return 0


if __name__ == "__main__":
    sys.exit(main())
