#!/usr/bin/env python
"""Benchmark of the two CLATCH hot paths on B200 (contract: see the task brief).

Workload = BASELINE.json configs[1] ("cfg2"): one 1920x1080 synthetic grayscale image,
10k oriented keypoints; a STEP = extract the 10k 512-bit descriptors + brute-force
10k x 10k Hamming top-2 self-match. The headline unit folds both halves of
BASELINE.json's metric into one number — keypoints/s, where one keypoint = one
descriptor extracted and its 10k Hamming compares matched — and the two halves are
also reported separately (descriptors/s, compares/s) from per-kernel CUDA events.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N>1 (under torchrun): every rank runs the same step on its own image (independent
units, no data-path collective) -> weak scaling; time = max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (width, height, keypoints, image seed, keypoint seed)   — SURVEY.md §8(d)
    "cfg1": (640, 480, 2000, 1609, 1610),
    "cfg2": (1920, 1080, 10000, 3986, 3987),
}
METRIC = ("descriptors/sec extracted and Hamming compares/sec matched "
          "(step = extract M descriptors + M x M Hamming top-2 match)")
UNIT = "keypoints/s (1 keypoint = 1 descriptor extracted + M Hamming compares)"

# Algorithmic work per unit.
FP64_OPS_PER_DESC = 4096 * 15 + 512 * 49 * 2 * 3          # non-fused fp64 ops (variants 0/1: everything in fp64)
SMEM_BYTES_PER_DESC = 512 * 49 * 3 * 8                     # 8-byte window reads in the SSD phase (variants 0/1)
# Variants 2/3 decide each bit from a proven fp32 estimate and recompute in fp64 only when undecided:
# the SSD phase reads 4-byte planes and runs fp32 FMAs; fp64 is left with the window resampling.
FILT_FP64_OPS_PER_DESC = 4096 * 15                         # resampling only
FILT_SMEM_BYTES_PER_DESC = 512 * 49 * 3 * 4                # 4-byte F-plane reads
POPC_PER_COMPARE = 16
# dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu --set full
# captures of the same command (profiles/*_ncu.json); cold-cache replay, so an upper bound.
TRAFFIC_NCU = {"extract_roles_kernel<16>": 2.419e+06,                # profiles/r2c_extract_ncu.json
               "extract_pipe_kernel": 2.419e+06,                     # profiles/r2c_extract_ncu.json
               "extract_quad_kernel<u8>": 2.419e+06,                 # profiles/r1t_extract_ncu.json
               "match_tc_kernel (tcgen05 kind::i8)": 5.288e+06}     # profiles/r2c_match_tc_ncu.json


def synth_inputs(workload: str, rank: int = 0):
    import oracle
    port = oracle.port()
    w, h, n, s_img, s_kp = WORKLOADS[workload]
    img = port.random_image_u8(s_img + 1000 * rank, w, h)
    kps = port.random_keypoints(s_kp + 1000 * rank, w, h, n)
    return img, kps


# ------------------------------------------------------------------ clocks ----

class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits", "-lms", "100",
                 "-i", str(self.index)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _pump(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            self.thread.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0])); mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for name, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)), "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------- reference arm ----

def cpu_step(img_f64, kps, threads: int, reps: int):
    """One cfg step on the host cores: the reference's describe_all + match_brute_force
    (oracle/_ref) or, without it, the C restatement threaded from here. Returns
    (seconds per step, t_describe, t_match, kind, descriptors)."""
    import oracle
    ref = oracle.ref()
    n = len(kps)
    if ref is not None:
        import ctypes as C
        L = ref.lib
        img = np.ascontiguousarray(img_f64)
        k = np.ascontiguousarray(kps)
        h, w = img.shape
        state = L.ref_bench_create(img.ctypes.data_as(oracle._f64p), w, h, k.ctypes.data_as(oracle._f64p), n)
        td = tm = 0.0
        m = 0
        for _ in range(reps):
            t0 = time.perf_counter()
            m = L.ref_bench_describe(state, n, threads)          # describe_all(..., workers)
            t1 = time.perf_counter()
            # gallery = probes (self-match): copy the descriptors the describe leg produced
            L.ref_bench_gallery_from_probes(state)
            t2 = time.perf_counter()
            cs = C.c_uint64()
            L.ref_bench_match(state, m, threads, C.byref(cs))     # match_brute_force(..., {workers})
            t3 = time.perf_counter()
            td += t1 - t0
            tm += t3 - t2
        L.ref_bench_destroy(state)
        return (td + tm) / reps, td / reps, tm / reps, "reference", m
    # port: thread the serial C restatement over contiguous chunks (ctypes drops the GIL)
    from concurrent.futures import ThreadPoolExecutor
    port = oracle.port()
    chunks = np.array_split(np.arange(n), threads)
    td = tm = 0.0
    for _ in range(reps):
        t0 = time.perf_counter()
        with ThreadPoolExecutor(threads) as ex:
            parts = list(ex.map(lambda c: port.describe_all(img_f64, kps[c])[1], chunks))
        desc = np.concatenate(parts)
        t1 = time.perf_counter()
        m = len(desc)
        bounds = np.linspace(0, m, threads + 1).astype(int)
        with ThreadPoolExecutor(threads) as ex:
            list(ex.map(lambda i: port.knn2_all(desc, desc, int(bounds[i]), int(bounds[i + 1])), range(threads)))
        t2 = time.perf_counter()
        td += t1 - t0
        tm += t2 - t1
    return (td + tm) / reps, td / reps, tm / reps, "port", m


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return                                  # other ranks exit 0 without work
    import oracle
    img, kps = synth_inputs(args.workload)
    threads = oracle.cpu_threads()
    img_f64 = img.astype(np.float64)
    for _ in range(args.warmup):
        cpu_step(img_f64, kps, threads, 1)
    t0 = time.perf_counter()
    td = tm = 0.0
    kind, m = "port", 0
    for _ in range(args.steps):
        _, d, mt, kind, m = cpu_step(img_f64, kps, threads, 1)
        td += d
        tm += mt
    elapsed = time.perf_counter() - t0
    per_step = elapsed / args.steps
    value = m / per_step
    w, h, n, _, _ = WORKLOADS[args.workload]
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64/u64-popcount",
        "data": "synthetic",
        "config": {"workload": f"{args.workload}: {w}x{h} u8-valued noise image, {n} oriented keypoints, "
                               f"extract + {m}x{m} top-2 self-match", "keypoints": n, "descriptors": m},
        "descriptors_per_s": m / (td / args.steps), "compares_per_s": m * m / (tm / args.steps),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": kind,
                         "sample": "the full step (describe_all + match_brute_force, workers = all host threads)"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    emit(line)


# ---------------------------------------------------------------- our arm ----

def load_peaks():
    peaks = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            peaks = {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
        except Exception:
            pass
    pp = ROOT / "profiles" / "pipe_peaks.json"
    if pp.exists():
        try:
            peaks["pipes"] = json.loads(pp.read_text())
        except Exception:
            pass
    return peaks


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_1609_03986_b200 as lk

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    use_dist = "RANK" in os.environ          # under torchrun (any world size) exercise the NCCL path
    if use_dist:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    eng = lk.get_engine(local)
    eng.set_pattern(None)
    if args.match_variant is not None:
        eng.set_option("match_variant", args.match_variant)
    if args.extract_variant is not None:
        eng.set_option("extract_variant", args.extract_variant)

    w, h, n, _, _ = WORKLOADS[args.workload]
    img, kps = synth_inputs(args.workload, rank)
    xycs, kept = eng.prepare_keypoints(kps, w, h)
    m = len(xycs)

    # ---- device-resident step: inputs already in HBM -------------------------------
    d_img = torch.from_numpy(img).to(dev)
    d_xycs = torch.from_numpy(xycs).to(dev)
    d_desc = torch.empty((m, 64), dtype=torch.uint8, device=dev)
    d_res = torch.empty((3, m), dtype=torch.int32, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)     # > 126 MB L2

    def step(ev=None):
        if ev: ev[0].record()
        if args.phase in ("both", "extract"):
            eng.extract_device(d_img, d_xycs, out=d_desc)
        if ev: ev[1].record()
        if args.phase in ("both", "match"):
            eng.match_top2_device(d_desc, d_desc, out=d_res)
        if ev: ev[2].record()

    if args.phase == "match":
        eng.extract_device(d_img, d_xycs, out=d_desc)
    for _ in range(args.warmup):
        step()
        flush.zero_()
    events = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(args.steps)]
    torch.cuda.synchronize()
    if use_dist:
        dist.barrier()
    launches0 = eng.launch_count
    with ClockSampler(local) as clocks:
        t_wall0 = time.perf_counter()
        for i in range(args.steps):
            step(events[i])
            flush.zero_()                     # L2 flush between steps, outside the event pairs
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        t_wall = time.perf_counter() - t_wall0
    launches = eng.launch_count - launches0
    t_ext = sum(e[0].elapsed_time(e[1]) for e in events) / 1e3
    t_mat = sum(e[1].elapsed_time(e[2]) for e in events) / 1e3
    t_dev = t_ext + t_mat
    if use_dist:
        t = torch.tensor([t_dev, t_ext, t_mat], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_dev, t_ext, t_mat = t.tolist()

    # ---- end to end through the reference-facing API, host buffers -----------------
    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    e2e = {}
    for tag, host_img in (("f64", pinned(img.astype(np.float64))), ("u8", pinned(img))):
        host_kps = pinned(kps)

        def api_step():
            kept_k, desc = lk.describe(host_img, host_kps)
            return lk.match(desc, desc)

        for _ in range(max(3, args.warmup)):
            api_step()
        torch.cuda.synchronize()
        if use_dist:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            out = api_step()
        torch.cuda.synchronize()
        t_api = time.perf_counter() - t0
        if use_dist:
            dist.barrier()
            tt = torch.tensor([t_api], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t_api = tt.item()
        e2e[tag] = {
            "value": world * m * args.steps / t_api, "unit": UNIT, "ms_per_step": t_api / args.steps * 1e3,
            "h2d_bytes_per_step": int(host_img.nbytes + m * 32 + m * 64),
            "d2h_bytes_per_step": int(m * 64 + 3 * 4 * m),
            "api": f"describe({tag} image (H,W), keypoints (N,4)) + match(desc, desc), pinned host arrays",
        }
        assert len(out) == m

    if rank != 0:
        if use_dist:
            dist.destroy_process_group()
        return

    # ---- reporting -------------------------------------------------------------------
    peaks = load_peaks()
    per_step = t_dev / args.steps
    ext_s, mat_s = t_ext / args.steps, t_mat / args.steps
    sm_mhz = clocks.summary()["sm_mhz"] or 1965.0
    sms = eng.sm_count
    pipes = peaks.get("pipes", {})
    mv = args.match_variant if args.match_variant is not None else 3
    ev = args.extract_variant if args.extract_variant is not None else 4
    ext_name = {0: "extract_fast_kernel<u8>", 1: "extract_quad_kernel<u8>", 2: "extract_filt_kernel",
                3: "extract_pipe_kernel", 4: "extract_roles_kernel<16>"}[ev]
    mat_name = "match_tc_kernel (tcgen05 kind::i8)" if mv == 3 else f"match64_kernel<{mv}>"
    kernels, pipe_roofline = {}, {}
    if ext_s > 0:
        alg_bytes = img.nbytes + m * 32 + m * 64            # image once + keypoint records + descriptors out
        filt = ev >= 2
        smem_bytes = FILT_SMEM_BYTES_PER_DESC if filt else SMEM_BYTES_PER_DESC
        smem_gbs = m * smem_bytes / ext_s / 1e9
        fp64_gops = m * (FILT_FP64_OPS_PER_DESC if filt else FP64_OPS_PER_DESC) / ext_s / 1e9
        kernels[ext_name] = {
            "ms": ext_s * 1e3, "descriptors_per_s": m / ext_s,
            "hbm": {"achieved": alg_bytes / ext_s / 1e9, "algorithmic_bytes_per_launch": alg_bytes},
            "fp64_gops": fp64_gops, "smem_gbs": smem_gbs,
        }
        smem_peak = pipes.get("lds64_gbs", sms * 128 * sm_mhz * 1e6 / 1e9)
        fp64_peak = pipes.get("fp64_nonfused_gops", sms * 64 * sm_mhz * 1e6 / 1e9)
        pipe_roofline["extract"] = {
            "bound": (f"shared-memory wavefronts ({smem_bytes // 1000} KB of {4 if filt else 8}-byte window reads per "
                      "descriptor" + ("; fp32 estimate + exact fp64 recompute of undecided bits)" if filt else ")")),
            "smem": {"achieved_gbs": smem_gbs, "peak_gbs": smem_peak, "frac": smem_gbs / smem_peak},
            "fp64": {"achieved_gops": fp64_gops, "peak_gops": fp64_peak, "frac": fp64_gops / fp64_peak},
            "peak_source": "measured microbench (profiles/pipe_peaks.json)" if pipes else
                           f"theoretical: {sms} SMs x 128 B/clk and x 64 lanes/clk at the sampled {sm_mhz:.0f} MHz",
        }
    if mat_s > 0:
        alg_bytes = 2 * m * 64 + 3 * 4 * m                  # both sets once + top-2 triples out
        cps = m * m / mat_s
        kernels[mat_name] = {
            "ms": mat_s * 1e3, "compares_per_s": cps,
            "hbm": {"achieved": alg_bytes / mat_s / 1e9, "algorithmic_bytes_per_launch": alg_bytes},
        }
        if mv == 3:
            # one compare = 512 int8 MACs = 1024 ops; int8 dense peak = 2 x the bf16 peak
            tops = cps * 1024 / 1e12
            bf16 = None
            try:
                bf16 = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"])
            except Exception:
                pass
            peak = 2 * bf16 if bf16 else 2 * 1590.0
            pipe_roofline["match"] = {
                "bound": "tensor", "achieved": tops, "peak": peak, "unit": "TOP/s (int8)", "frac": tops / peak,
                "peak_source": ("2 x measured bf16 burst GEMM peak (MEASURED_PEAKS.json); nominal int8 dense 4500"
                                if bf16 else "2 x fallback bf16 peak"),
                "includes": "bit->int8 expansion of both sets, the GEMM + top-2 epilogue, and the split merge",
            }
        else:
            popc = {0: 16, 1: 9, 2: 7}[mv]
            popc_peak = pipes.get("popc_gops", sms * 16 * sm_mhz * 1e6 / 1e9)
            pipe_roofline["match"] = {
                "bound": "popc (XU pipe)", "achieved_gops": cps * popc / 1e9, "peak_gops": popc_peak,
                "frac": cps * popc / 1e9 / popc_peak, "popc_per_compare": popc,
                "peak_source": "measured microbench (profiles/pipe_peaks.json)" if pipes else
                               f"theoretical: {sms} SMs x 16 POPC/clk at the sampled {sm_mhz:.0f} MHz",
            }
    dom = max(kernels, key=lambda k: kernels[k]["ms"])
    roofline = {
        "kernel": dom, "bound": "hbm", "achieved": kernels[dom]["hbm"]["achieved"], "peak": peaks["hbm_gbs"],
        "unit": "GB/s", "frac": kernels[dom]["hbm"]["achieved"] / peaks["hbm_gbs"], "peak_source": peaks["source"],
        "traffic": TRAFFIC_NCU.get(dom),
        "note": "contract form (algorithmic HBM bytes / kernel time). Neither kernel is HBM-bound "
                "(SURVEY.md 8d): the binding resources and their fractions are in 'pipe_roofline'",
    }

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        import oracle
        threads = oracle.cpu_threads()
        sec, td, tm, kind, mm = cpu_step(img.astype(np.float64), kps, threads, 2)
        cpu = {"value": mm / sec, "unit": UNIT, "cores": threads, "kind": kind,
               "sample": "the full step twice (describe_all + match_brute_force, workers = all host threads)",
               "descriptors_per_s": mm / td, "compares_per_s": mm * mm / tm}

    dtype = ("f64 resampling, " + ("fp32 estimate + exact f64 recompute" if ev >= 2 else "f64 SSD") + " (extraction) / " +
             ("int8 tcgen05, int32 accumulate" if mv == 3 else "u32 xor+popc") + " (matching); results bit-exact")
    line = {
        "metric": METRIC, "value": world * m / per_step, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": dtype, "data": "synthetic",
        "config": {"workload": f"{args.workload}: {w}x{h} u8 noise image, {n} oriented keypoints per GPU, "
                               f"extract + {m}x{m} Hamming top-2 self-match", "keypoints": n, "descriptors": m,
                   "phase": args.phase,
                   "l2": "256 MiB device memset between steps, outside the per-step CUDA-event pairs",
                   "timing": "sum of per-step CUDA-event durations on the launching stream, max over ranks"},
        "descriptors_per_s": world * m / ext_s if ext_s > 0 else None,
        "compares_per_s": world * m * m / mat_s if mat_s > 0 else None,
        "wall_ms_per_step_incl_flush": t_wall / args.steps * 1e3,
        "clocks": clocks.summary(), "e2e": e2e["f64"], "e2e_u8": e2e["u8"], "gpu_launches": int(launches),
        "roofline": roofline, "pipe_roofline": pipe_roofline, "kernels": kernels, "cpu_baseline": cpu,
        "device": eng.name, "sm_count": sms,
    }
    emit(line)
    if use_dist:
        dist.destroy_process_group()


# stdout carries exactly ONE JSON line. Libraries write there too (NCCL prints its version line at
# every NCCL_DEBUG level from WARN up, straight from C): everything else is pointed at stderr for the
# whole run and the line goes out through a private duplicate of the original descriptor.
_JSON_FD = None


def capture_stdout():
    global _JSON_FD
    if _JSON_FD is None:
        sys.stdout.flush()
        _JSON_FD = os.dup(1)
        os.dup2(2, 1)


def emit(line: dict):
    data = (json.dumps(line) + "\n").encode()
    if _JSON_FD is None:
        sys.stdout.write(data.decode())
        sys.stdout.flush()
    else:
        os.write(_JSON_FD, data)


def main():
    capture_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="cfg2")
    ap.add_argument("--phase", choices=["both", "extract", "match"], default="both")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--match-variant", type=int, default=None, help="override the matcher kernel variant (0..4)")
    ap.add_argument("--extract-variant", type=int, default=None, help="override the extraction kernel variant (0..4)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
