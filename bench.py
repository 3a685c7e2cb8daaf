#!/usr/bin/env python
"""Benchmark of the two CLATCH hot paths on B200 (contract: see the task brief).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload cfgK|all]

BASELINE.json names five configurations (oracle/workloads.py draws their inputs with the
reference's generator and the seeds of SURVEY.md §8d):

    cfg1  640x480, 2 000 keypoints: extract + 2k x 2k top-2 self-match
    cfg2  1920x1080, 10 000 keypoints: extract + 10k x 10k            <- the headline, configs[1]
    cfg3  64 images 3840x2160 x 50 000 keypoints: extraction, sharded by image
    cfg4  1 M x 1 M descriptors, ratio 0.8: train set broadcast, queries sharded
    cfg5  256 images x 8 000 keypoints: all 32 640 image pairs (ratio 0.8 + cross-check), pairs sharded

Default (`--workload all`): the line's headline (`value`, `e2e`, `roofline`, `cpu_baseline`) is the
cfg2 step — at N > 1 one step per rank on its own image, no data-path collective, max over ranks —
and `configs` carries one sub-record per configuration, cfg3/4/5 at FULL size through
paper_1609_03986_b200/sharded.py (strong scaling: the job is fixed, the ranks split it; NCCL under
torchrun at any world size). `--workload cfgK` makes that configuration the headline instead.
The headline workload is the same at every N because the driver derives scaling efficiency from
`value` across N; the sharded configurations' strong-scaling numbers ride along in `configs`.

`--impl reference`: the unmodified reference (oracle/_ref, else the C restatement) on the host
cores, same configuration strings; the big configurations run the bounded samples of BASELINE.md §3.
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

METRIC = ("descriptors/sec extracted and Hamming compares/sec matched "
          "(step = extract M descriptors + M x M Hamming top-2 match)")
UNIT = "keypoints/s (1 keypoint = 1 descriptor extracted + M Hamming compares)"
UNITS = {"cfg1": UNIT, "cfg2": UNIT, "cfg3": "descriptors/s", "cfg4": "Hamming compares/s",
         "cfg5": "image pairs/s (1 pair = 8000 x 8000 top-2 forward + reverse + filter pass)"}
METRICS = {"cfg1": METRIC, "cfg2": METRIC,
           "cfg3": "descriptors/sec extracted (64 images x 50 000 keypoints, sharded by image)",
           "cfg4": "Hamming compares/sec matched (1 M x 1 M top-2 + ratio test, queries sharded)",
           "cfg5": "image pairs/sec matched (all pairs of 256 descriptor sets, ratio test + cross-check, pairs sharded)"}

# Algorithmic work per unit.
FP64_OPS_PER_DESC = 4096 * 15 + 512 * 49 * 2 * 3          # non-fused fp64 ops (variants 0/1: everything in fp64)
SMEM_BYTES_PER_DESC = 512 * 49 * 3 * 8                     # 8-byte window reads in the SSD phase (variants 0/1)
# Variants 2-4 decide each bit from a proven fp32 estimate and recompute in fp64 only when undecided:
# the SSD phase reads 4-byte planes and runs fp32 FMAs; fp64 is left with the window resampling.
FILT_FP64_OPS_PER_DESC = 4096 * 15                         # resampling only
FILT_SMEM_BYTES_PER_DESC = 512 * 49 * 3 * 4                # 4-byte F-plane reads
# variants 5 / 6: the planes hold 16-bit samples in two shifted copies; a 7-pixel patch row is four aligned 32-bit words,
# and the resampling runs in fp32 (fp64 only sets up each thread's start coordinates, 12 ops per thread and window).
H16_SMEM_BYTES_PER_DESC = 512 * 7 * 4 * 3 * 4              # 28 word loads per patch
H16_FP64_OPS_PER_DESC = 512 * 12 + 64
# ... and what binds them is the issue rate (ncu: issue slots 70 % busy, shared-memory pipe 59 %, ALU pipe 52 %). Algorithmic
# warp instructions per descriptor: estimate = 256 slot pairs x 49 pixels x (6 unpacks + 4 packed FMAs + 6 * 28/49 loads) / 32
# lanes = 5 264; resampling = 4 096 samples x 23.5 (coordinates 10, gather 1, three lerps 6, round 1, pack + stores 2.5,
# steps 3) / 32 = 3 008. Peak: one warp instruction per clock and scheduler, 4 schedulers per SM.
H16_WARP_INSTR_PER_DESC = 5264 + 3008
INT8_OPS_PER_COMPARE = 1024                                # 512 int8 MACs
EXTRACT_KERNELS = {0: "extract_fast_kernel<u8>", 1: "extract_quad_kernel<u8>", 2: "extract_filt_kernel",
                   3: "extract_pipe_kernel", 4: "extract_roles_kernel<16>", 5: "extract_h16_kernel<16, false>", 6: "extract_h16s_kernel"}
# committed ncu --set full captures (tools/summarize_ncu.py), newest visit first; `traffic` is read from these files
NCU_PROFILES = {"extract": ("r*_extract_ncu.json", "extract_"), "match": ("r*_match_tc_ncu.json", "match_tc")}


def wl():
    import oracle.workloads as w          # input synthesis + CPU baseline only; never on the timed GPU path
    return w


def synth_inputs(workload: str, rank: int = 0):
    """(u8 image, keypoints) of an image configuration — kept for the tools/ scripts."""
    W = wl()
    return W.image(workload, 0, rank), W.keypoints(workload, 0, rank)


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


# ------------------------------------------------------- CPU / reference legs ----

def cpu_image_step(img_f64, kps, threads: int, reps: int):
    """One cfg1/cfg2 step on the host cores: the reference's describe_all + match_brute_force
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
            L.ref_bench_gallery_from_probes(state)               # self-match: gallery = the probes just made
            t2 = time.perf_counter()
            cs = C.c_uint64()
            L.ref_bench_match(state, m, threads, C.byref(cs))     # match_brute_force(..., {workers})
            t3 = time.perf_counter()
            td += t1 - t0
            tm += t3 - t2
        L.ref_bench_destroy(state)
        return (td + tm) / reps, td / reps, tm / reps, "reference", m
    W = wl()
    td = tm = 0.0
    m = 0
    for _ in range(reps):
        t0 = time.perf_counter()
        desc = W.describe_all_threaded(img_f64, kps, threads)[1]
        t1 = time.perf_counter()
        W.knn2_rows_threaded(desc, desc, threads)
        t2 = time.perf_counter()
        td += t1 - t0
        tm += t2 - t1
        m = len(desc)
    return (td + tm) / reps, td / reps, tm / reps, "port", m


def cpu_sample(cfg: str, threads: int):
    """One bounded sample of a configuration on the host cores -> dict with the
    whole-job value in the configuration's unit. Reference build when oracle/_ref exists."""
    import oracle
    W = wl()
    ref = oracle.ref()
    kind = "reference" if ref is not None else "port"
    if cfg in ("cfg1", "cfg2"):
        img = W.image(cfg).astype(np.float64)
        kps = W.keypoints(cfg)
        sec, td, tm, kind, m = cpu_image_step(img, kps, threads, 1)
        return {"value": m / sec, "unit": UNITS[cfg], "cores": threads, "kind": kind, "seconds": sec,
                "sample": "the full step (describe_all + match_brute_force, workers = all host threads)",
                "descriptors_per_s": m / td, "compares_per_s": m * m / tm}

    def describe(img, kps):
        if ref is not None:
            return ref.describe_all(img, kps, workers=threads)[1]
        return W.describe_all_threaded(img, kps, threads)[1]

    def match(a, b, **kw):
        if ref is not None:
            return ref.match(a, b, workers=threads, **kw)
        return W.match_threaded(a, b, threads=threads, **kw)

    if cfg == "cfg3":
        imgs, kps = W.images_and_keypoints("cfg3", range(2))
        t0 = time.perf_counter()
        m = sum(len(describe(im.astype(np.float64), k)) for im, k in zip(imgs, kps))
        sec = time.perf_counter() - t0
        return {"value": m / sec, "unit": UNITS[cfg], "cores": threads, "kind": kind, "seconds": sec,
                "sample": "describe_all on 2 of the 64 images (100 000 keypoints), workers = all host threads; "
                          "the 64-image job is 32x this"}
    if cfg == "cfg4":
        q, t, _ = W.cfg4_sets()
        rows = 4096
        t0 = time.perf_counter()
        match(q[:rows], t, ratio=W.RATIO)
        sec = time.perf_counter() - t0
        return {"value": rows * len(t) / sec, "unit": UNITS[cfg], "cores": threads, "kind": kind, "seconds": sec,
                "sample": f"match_brute_force(ratio 0.8) of the first {rows} query rows against the full 1 M train set, "
                          "workers = all host threads; the job is 244x this"}
    if cfg == "cfg5":
        imgs, kps = W.images_and_keypoints("cfg5", range(9))
        t0 = time.perf_counter()
        sets = [describe(im.astype(np.float64), k) for im, k in zip(imgs[:2], kps[:2])]
        t_img = (time.perf_counter() - t0) / 2
        # descriptor sets for the pair sample: the remaining images come from the C restatement (untimed)
        sets += [W.describe_all_threaded(im, k, threads)[1] for im, k in zip(imgs[2:], kps[2:])]
        t0 = time.perf_counter()
        for j in range(1, 9):
            match(sets[0], sets[j], ratio=W.RATIO, cross_check=True)
        t_pair = (time.perf_counter() - t0) / 8
        n_img = W.IMAGE_CONFIGS["cfg5"][5]
        n_pairs = n_img * (n_img - 1) // 2
        return {"value": n_pairs / (n_img * t_img + n_pairs * t_pair), "unit": UNITS[cfg], "cores": threads,
                "kind": kind, "seconds": 2 * t_img + 8 * t_pair, "s_per_image": t_img, "s_per_pair": t_pair,
                "sample": "describe_all on 2 images + match_brute_force(ratio 0.8, cross_check) on 8 image pairs, "
                          "workers = all host threads; whole job extrapolated as 256 images + 32 640 pairs"}
    raise ValueError(cfg)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return                                  # other ranks exit 0 without work
    import oracle
    W = wl()
    threads = oracle.cpu_threads()
    head = "cfg2" if args.workload == "all" else args.workload
    extra = {}
    if head in ("cfg1", "cfg2"):
        img = W.image(head).astype(np.float64)
        kps = W.keypoints(head)
        for _ in range(args.warmup):
            cpu_image_step(img, kps, threads, 1)
        t0 = time.perf_counter()
        td = tm = 0.0
        kind, m = "port", 0
        for _ in range(args.steps):
            _, d, mt, kind, m = cpu_image_step(img, kps, threads, 1)
            td += d
            tm += mt
        per_step = (time.perf_counter() - t0) / args.steps
        value = m / per_step
        sample = "the full step (describe_all + match_brute_force, workers = all host threads)"
        extra = {"descriptors_per_s": m / (td / args.steps), "compares_per_s": m * m / (tm / args.steps)}
    else:
        for _ in range(min(args.warmup, 1)):
            cpu_sample(head, threads)
        vals, secs = [], []
        for _ in range(args.steps):
            s = cpu_sample(head, threads)
            vals.append(s["value"]); secs.append(s["seconds"])
        value, per_step, kind, sample = float(np.mean(vals)), float(np.mean(secs)), s["kind"], s["sample"]
    line = {
        "impl": "reference", "metric": METRICS[head], "value": value, "unit": UNITS[head], "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3,
        "higher_is_better": True, "scaling": "weak" if head in ("cfg1", "cfg2") else "strong", "vs_baseline": None,
        "dtype": "f64/u64-popcount", "data": "synthetic", "config": {"workload": W.DESCRIPTIONS[head]},
        "cpu_baseline": {"value": value, "unit": UNITS[head], "cores": threads, "kind": kind, "sample": sample},
        "e2e": {"value": value, "unit": UNITS[head], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0, **extra,
    }
    if args.workload == "all":
        configs = {}
        for cfg in ("cfg1", "cfg3", "cfg4", "cfg5"):
            s = cpu_sample(cfg, threads)
            configs[cfg] = {"workload": W.DESCRIPTIONS[cfg], **s}
        configs["cfg2"] = {"workload": W.DESCRIPTIONS["cfg2"], "value": value, "unit": UNIT, "cores": threads,
                           "kind": kind, "sample": sample}
        line["configs"] = dict(sorted(configs.items()))
    emit(line)


# ---------------------------------------------------------------- our arm ----

def load_peaks():
    peaks = {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)", "bf16_tflops": None}
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            peaks.update(hbm_gbs=float(d["hbm_gbs"]), source="measured (MEASURED_PEAKS.json)",
                         bf16_tflops=float(d["bf16_tflops"]), bf16_sustained=float(d.get("bf16_tflops_sustained", 0)) or None)
        except Exception:
            pass
    pp = ROOT / "profiles" / "pipe_peaks.json"
    if pp.exists():
        try:
            peaks["pipes"] = json.loads(pp.read_text())
        except Exception:
            pass
    return peaks


def ncu_traffic(which: str, kernel: str | None = None):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of the dominant kernel, from the committed
    `ncu --set full` capture of this command (cold-cache replay, so an upper bound). None if absent."""
    pattern, prefix = NCU_PROFILES[which]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for path in sorted((ROOT / "profiles").glob(pattern), reverse=True):
        try:
            rows = json.loads(path.read_text())
        except Exception:
            continue
        for r in rows:
            if prefix in r.get("kernel", "") and (kernel is None or kernel.split("<")[0] in r["kernel"]):
                tot = 0.0
                for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    tot += float(r.get(k, 0.0)) * scale.get(r.get(k + " [unit]", "byte"), 1.0)
                return tot, f"profiles/{path.name}"
    return None, None


class Ctx:
    """What every configuration runner needs: the engine, torch device, rank layout and timing helpers."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist

        import paper_1609_03986_b200 as lk
        self.torch, self.dist, self.lk, self.args = torch, dist, lk, args
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        self.use_dist = "RANK" in os.environ     # under torchrun (any world size) exercise the NCCL path
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.use_dist:
            dist.init_process_group("nccl", device_id=self.dev)
        os.environ.setdefault("CLATCH_DEVICE", str(self.local))
        self.eng = lk.get_engine(self.local)
        self.eng.set_pattern(None)
        if args.match_variant is not None:
            self.eng.set_option("match_variant", args.match_variant)
        if args.extract_variant is not None:
            self.eng.set_option("extract_variant", args.extract_variant)
        self.flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device=self.dev)     # > 126 MB L2
        self.peaks = load_peaks()
        self.mv = args.match_variant if args.match_variant is not None else 4
        self.ev = args.extract_variant if args.extract_variant is not None else 5

    def flush(self):
        self.flush_buf.zero_()

    def sync(self):
        self.torch.cuda.synchronize()
        self.eng.synchronize()

    def barrier(self):
        self.sync()
        if self.use_dist:
            self.dist.barrier()

    def max_over_ranks(self, *vals):
        if not self.use_dist:
            return list(vals)
        t = self.torch.tensor(vals, dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return t.tolist()

    def sum_over_ranks(self, *vals):
        if not self.use_dist:
            return list(vals)
        t = self.torch.tensor(vals, dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t)
        return t.tolist()

    def pinned(self, a: np.ndarray) -> np.ndarray:
        t = self.torch.empty(a.shape, dtype=self.torch.from_numpy(a[:0]).dtype, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    def time_events(self, step, steps, warmup, marks=2):
        """`step(ev)` records ev[0..marks-1] on torch's current stream (the kernels' launching stream).
        Returns per-interval device seconds summed over the timed steps, max over ranks; L2 is flushed
        between steps outside the event pairs."""
        torch = self.torch
        for _ in range(warmup):
            step(None)
            self.flush()
        events = [[torch.cuda.Event(enable_timing=True) for _ in range(marks)] for _ in range(steps)]
        self.barrier()
        t0 = time.perf_counter()
        for i in range(steps):
            step(events[i])
            self.flush()
        self.barrier()
        wall = time.perf_counter() - t0
        spans = [sum(e[k].elapsed_time(e[k + 1]) for e in events) / 1e3 for k in range(marks - 1)]
        return self.max_over_ranks(*spans), wall

    def time_wall(self, fn, steps, warmup):
        """Host-clock timing of a synchronous API call (sync + barrier on both sides), max over ranks.
        Returns (seconds per step, last result)."""
        out = None
        for _ in range(warmup):
            out = fn()
            self.flush()
        self.barrier()
        total = 0.0
        for _ in range(steps):
            self.sync()
            t0 = time.perf_counter()
            out = fn()
            self.sync()
            total += time.perf_counter() - t0
            self.flush()
        self.barrier()
        return self.max_over_ranks(total / steps)[0], out

    # ---- rooflines ----
    def extract_roofline(self, descriptors: float, seconds: float, sm_mhz: float, hbm_bytes: float):
        pipes = self.peaks.get("pipes", {})
        sms = self.eng.sm_count
        filt = self.ev >= 2
        h16 = self.ev >= 5
        smem_bytes = H16_SMEM_BYTES_PER_DESC if h16 else FILT_SMEM_BYTES_PER_DESC if filt else SMEM_BYTES_PER_DESC
        fp64_ops = H16_FP64_OPS_PER_DESC if h16 else FILT_FP64_OPS_PER_DESC if filt else FP64_OPS_PER_DESC
        smem_gbs = descriptors * smem_bytes / seconds / 1e9
        fp64_gops = descriptors * fp64_ops / seconds / 1e9
        smem_peak = pipes.get("lds64_gbs", sms * 128 * sm_mhz * 1e6 / 1e9)
        fp64_peak = pipes.get("fp64_nonfused_gops", sms * 64 * sm_mhz * 1e6 / 1e9)
        traffic, src = ncu_traffic("extract", EXTRACT_KERNELS[self.ev])
        smem = {"bound": "smem", "achieved": smem_gbs, "peak": smem_peak, "unit": "GB/s", "frac": smem_gbs / smem_peak,
                "algorithmic_bytes_per_descriptor": smem_bytes}
        if h16:
            issue_peak = sms * 4 * sm_mhz * 1e6 / 1e9                       # G warp-instructions / s
            issue = descriptors * H16_WARP_INSTR_PER_DESC / seconds / 1e9
            return {
                "kernel": EXTRACT_KERNELS[self.ev], "bound": "issue", "achieved": issue, "peak": issue_peak,
                "unit": "G warp-instr/s", "frac": issue / issue_peak,
                "what": f"instruction issue: {H16_WARP_INSTR_PER_DESC} algorithmic warp instructions per descriptor (estimate 5264: "
                        "256 slot pairs x 49 pixels x (6 PRMT unpacks + 4 FFMA2 + 3.43 LDS) / 32; resampling 3008: 4096 samples x "
                        "23.5 / 32) x descriptors per launch / kernel time. ncu on this kernel: issue slots 70 % busy, "
                        "shared-memory pipe 59 %, ALU pipe 52 % — the issue rate binds, not a data path",
                "peak_source": f"{sms} SMs x 4 schedulers x 1 warp instruction / clk at the sampled {sm_mhz:.0f} MHz",
                "traffic": traffic, "traffic_source": src, "smem": smem,
                "fp64": {"achieved_gops": fp64_gops, "peak_gops": fp64_peak, "frac": fp64_gops / fp64_peak},
                "hbm": {"bound": "hbm", "achieved": hbm_bytes / seconds / 1e9, "peak": self.peaks["hbm_gbs"], "unit": "GB/s",
                        "frac": hbm_bytes / seconds / 1e9 / self.peaks["hbm_gbs"], "algorithmic_bytes": hbm_bytes,
                        "peak_source": self.peaks["source"],
                        "note": "contract form (image + keypoint records + descriptors once); HBM does not bind this kernel"},
            }
        return {
            "kernel": EXTRACT_KERNELS[self.ev], "bound": "smem", "achieved": smem_gbs, "peak": smem_peak, "unit": "GB/s",
            "frac": smem_gbs / smem_peak,
            "what": (f"shared-memory wavefronts: {smem_bytes} B of 4-byte plane reads per descriptor (512 triplets x 3 patches x "
                     "7 rows x 4 aligned words of packed 16-bit samples) x descriptors per launch / kernel time") if h16 else
                    (f"shared-memory wavefronts: {smem_bytes} B of {4 if filt else 8}-byte window reads per descriptor "
                     "(512 triplets x 49 live pixels x 3 patches) x descriptors per launch / kernel time"),
            "peak_source": ("measured microbench: conflict-free 64-bit shared loads, tools/pipe_peaks.cu -> "
                            "profiles/pipe_peaks.json") if pipes else
                           f"theoretical: {sms} SMs x 128 B/clk at the sampled {sm_mhz:.0f} MHz",
            "traffic": traffic, "traffic_source": src,
            "fp64": {"achieved_gops": fp64_gops, "peak_gops": fp64_peak, "frac": fp64_gops / fp64_peak},
            "hbm": {"bound": "hbm", "achieved": hbm_bytes / seconds / 1e9, "peak": self.peaks["hbm_gbs"], "unit": "GB/s",
                    "frac": hbm_bytes / seconds / 1e9 / self.peaks["hbm_gbs"], "algorithmic_bytes": hbm_bytes,
                    "peak_source": self.peaks["source"],
                    "note": "contract form (image + keypoint records + descriptors once); HBM does not bind this kernel"},
        }

    def match_roofline(self, compares: float, seconds: float, sm_mhz: float, hbm_bytes: float, includes: str):
        pipes = self.peaks.get("pipes", {})
        sms = self.eng.sm_count
        cps = compares / seconds
        hbm = {"bound": "hbm", "achieved": hbm_bytes / seconds / 1e9, "peak": self.peaks["hbm_gbs"], "unit": "GB/s",
               "frac": hbm_bytes / seconds / 1e9 / self.peaks["hbm_gbs"], "algorithmic_bytes": hbm_bytes,
               "peak_source": self.peaks["source"],
               "note": "contract form (both sets + top-2 triples once); HBM does not bind this kernel"}
        if self.mv in (3, 4):
            tops = cps * INT8_OPS_PER_COMPARE / 1e12
            key, kind = ("mxf4", "kind::mxf4 e2m1, f32 accumulate") if self.mv == 4 else ("int8", "kind::i8, int32 accumulate")
            if pipes.get(key + "_tops"):
                peak = float(pipes[key + "_tops"])
                src = (f"measured: tcgen05 {kind}, M128 N256 issue loop without epilogue at {pipes.get(key + '_sm_mhz')} MHz "
                       "(tools/tc_peak.cu -> profiles/pipe_peaks.json); under the power cap of a long run the clock, and with "
                       "it this peak, drops — see 'clock_scaled'")
            elif self.peaks.get("bf16_tflops"):
                peak, src = (4 if self.mv == 4 else 2) * self.peaks["bf16_tflops"], "bf16 burst GEMM peak (MEASURED_PEAKS.json) x 2 (int8) or x 4 (fp4)"
            else:
                peak, src = (4 if self.mv == 4 else 2) * 1590.0, "fallback bf16 peak x 2 (int8) or x 4 (fp4)"
            traffic, tsrc = ncu_traffic("match")
            per_clk = float(pipes.get(key + "_mac_per_clk_sm", 16384 if self.mv == 4 else 8192))
            scaled = 2 * per_clk * sms * sm_mhz * 1e6 / 1e12      # the same pipe at the clock sampled during THIS run
            return {"kernel": f"match_tc_kernel (tcgen05 {kind})", "bound": "tensor", "achieved": tops, "peak": peak,
                    "unit": "TOP/s (1 compare = 512 MACs = 1024 ops)", "frac": tops / peak, "peak_source": src,
                    "clock_scaled": {"sm_mhz": sm_mhz, "peak": scaled, "frac": tops / scaled,
                                     "note": "MACs/clk/SM of the microbenchmark x SMs x the SM clock sampled during this run"},
                    "includes": includes, "traffic": traffic, "traffic_source": tsrc, "hbm": hbm}
        popc = {0: 16, 1: 9, 2: 7}[self.mv]
        popc_peak = pipes.get("popc_gops", sms * 16 * sm_mhz * 1e6 / 1e9)
        return {"kernel": f"match64_kernel<{self.mv}>", "bound": "popc (XU pipe)", "achieved": cps * popc / 1e9,
                "peak": popc_peak, "unit": "GPOPC/s", "frac": cps * popc / 1e9 / popc_peak, "popc_per_compare": popc,
                "traffic": None, "hbm": hbm}


def run_image_step(cx: Ctx, cfg: str, steps: int, warmup: int, cpu: bool, clocks_out: dict):
    """cfg1 / cfg2: one image, extract + M x M top-2 self-match. N > 1: one step per rank on its own
    image (independent units, no data-path collective) -> weak scaling."""
    torch, eng, lk, args = cx.torch, cx.eng, cx.lk, cx.args
    W = wl()
    w, h, n = W.IMAGE_CONFIGS[cfg][:3]
    img, kps = W.image(cfg, 0, cx.rank), W.keypoints(cfg, 0, cx.rank)
    xycs, kept = eng.prepare_keypoints(kps, w, h)
    m = len(xycs)
    d_img = torch.from_numpy(img).to(cx.dev)
    d_xycs = torch.from_numpy(xycs).to(cx.dev)
    d_desc = torch.empty((m, 64), dtype=torch.uint8, device=cx.dev)
    d_res = torch.empty((3, m), dtype=torch.int32, device=cx.dev)

    def step(ev):
        if ev: ev[0].record()
        if args.phase in ("both", "extract"):
            eng.extract_device(d_img, d_xycs, out=d_desc)
        if ev: ev[1].record()
        if args.phase in ("both", "match"):
            eng.match_top2_device(d_desc, d_desc, out=d_res)
        if ev: ev[2].record()

    if args.phase == "match":
        eng.extract_device(d_img, d_xycs, out=d_desc)
    launches0 = eng.launch_count
    with ClockSampler(cx.local) as clocks:
        (t_ext, t_mat), wall = cx.time_events(step, steps, warmup, marks=3)
    launches = (eng.launch_count - launches0) * steps // (steps + warmup)
    clocks_out.update(clocks.summary())
    sm_mhz = clocks_out.get("sm_mhz") or 1965.0

    # ---- end to end through the reference-facing API, host buffers -----------------
    def e2e_leg(host_img, host_kps, tag, memory):
        def api_step():
            kept_k, desc = lk.describe(host_img, host_kps)
            return lk.match(desc, desc)
        sec, out = cx.time_wall(api_step, steps, max(3, warmup))
        assert len(out) == m
        return {"value": cx.world * m / sec, "unit": UNIT, "ms_per_step": sec * 1e3,
                "h2d_bytes_per_step": int(host_img.nbytes + m * 32 + m * 64),
                "d2h_bytes_per_step": int(m * 64 + 3 * 4 * m),
                "api": f"describe({tag} image (H,W), keypoints (N,4)) + match(desc, desc), {memory} host arrays"}

    img64 = img.astype(np.float64)
    e2e = e2e_leg(cx.pinned(img64), cx.pinned(kps), "f64", "page-locked")
    e2e_pageable = e2e_leg(img64, kps.copy(), "f64", "ordinary (pageable) numpy")
    e2e_u8 = e2e_leg(cx.pinned(img), cx.pinned(kps), "u8", "page-locked")
    # ... and a float64 frame that is NOT u8-valued (a warped / noisy frame): the float-texture route of the default kernel
    frac = img64 * 0.93 + np.random.default_rng(3988).random(img64.shape) * 3.0
    m_saved, m = m, len(lk.describe(frac, kps)[1])
    e2e_frac = e2e_leg(cx.pinned(frac), cx.pinned(kps), "non-integer f64", "page-locked")
    m = m_saved

    per_step = (t_ext + t_mat) / steps
    ext_s, mat_s = t_ext / steps, t_mat / steps
    kernels, roofs = {}, {}
    if ext_s > 0:
        roofs["extract"] = cx.extract_roofline(m, ext_s, sm_mhz, img.nbytes + m * 32 + m * 64)
        kernels[roofs["extract"]["kernel"]] = {"ms": ext_s * 1e3, "descriptors_per_s": m / ext_s}
    if mat_s > 0:
        roofs["match"] = cx.match_roofline(m * m, mat_s, sm_mhz, 2 * m * 64 + 12 * m,
                                           "bit->int8 expansion of both sets, the GEMM + top-2 epilogue, and the split merge")
        kernels[roofs["match"]["kernel"]] = {"ms": mat_s * 1e3, "compares_per_s": m * m / mat_s}
    dom = "extract" if ext_s >= mat_s else "match"
    roofline = dict(roofs[dom])
    roofline["other_kernel"] = {k: v for k, v in roofs.items() if k != dom}
    rec = {
        "workload": W.DESCRIPTIONS[cfg], "value": cx.world * m / per_step, "unit": UNIT, "ms_per_step": per_step * 1e3,
        "steps": steps, "warmup": warmup, "scaling": "weak",
        "descriptors_per_s": cx.world * m / ext_s if ext_s > 0 else None,
        "compares_per_s": cx.world * m * m / mat_s if mat_s > 0 else None,
        "wall_ms_per_step_incl_flush": wall / steps * 1e3,
        "e2e": e2e, "e2e_pageable": e2e_pageable, "e2e_u8": e2e_u8, "e2e_noninteger_f64": e2e_frac, "gpu_launches": int(launches),
        "roofline": roofline, "kernels": kernels, "keypoints": n, "descriptors": m,
        "timing": "sum of per-step CUDA-event durations on the launching stream, max over ranks; "
                  "256 MiB device memset between steps, outside the event pairs",
    }
    if cpu and cx.rank == 0 and cx.world == 1:
        import oracle
        threads = oracle.cpu_threads()
        sec, td, tm, kind, mm = cpu_image_step(img64, kps, threads, 2)
        rec["cpu_baseline"] = {"value": mm / sec, "unit": UNIT, "cores": threads, "kind": kind,
                               "sample": "the full step twice (describe_all + match_brute_force, workers = all host threads)",
                               "descriptors_per_s": mm / td, "compares_per_s": mm * mm / tm}
    return rec


def run_cfg3(cx: Ctx, steps: int, warmup: int, cpu: bool, clocks_out: dict):
    """64 images 3840x2160 x 50 000 keypoints, sharded by image (image i -> rank i mod world)."""
    torch, eng, lk = cx.torch, cx.eng, cx.lk
    from paper_1609_03986_b200 import sharded
    W = wl()
    w, h, n, _, _, count = W.IMAGE_CONFIGS["cfg3"]
    mine = list(range(cx.rank, count, cx.world))
    imgs, kps = W.images_and_keypoints("cfg3", mine)
    recs = [eng.prepare_keypoints(k, w, h)[0] for k in kps]
    d_imgs = [torch.from_numpy(a).to(cx.dev) for a in imgs]
    d_recs = [torch.from_numpy(r).to(cx.dev) for r in recs]
    d_out = [torch.empty((len(r), 64), dtype=torch.uint8, device=cx.dev) for r in recs]
    m_local = sum(len(r) for r in recs)
    m_total = int(cx.sum_over_ranks(m_local)[0])

    def step(ev):
        if ev: ev[0].record()
        for a, r, o in zip(d_imgs, d_recs, d_out):
            eng.extract_device(a, r, out=o)
        if ev: ev[1].record()

    launches0 = eng.launch_count
    with ClockSampler(cx.local) as clocks:
        (t_dev,), _ = cx.time_events(step, steps, warmup)
    launches = (eng.launch_count - launches0) * steps // (steps + warmup)
    clocks_out.update(clocks.summary())
    sec = t_dev / steps
    del d_imgs, d_recs, d_out

    full = [None] * count                 # extract_images_sharded reads only this rank's entries

    def e2e_leg(host_imgs, tag, memory):
        li, lk_ = list(full), list(full)
        for i, a, k in zip(mine, host_imgs, kps):
            li[i], lk_[i] = a, k
        # (warm-up >= 5: the page-locked result pool grows by one round of blocks per call that releases its results)
        s, out = cx.time_wall(lambda: sharded.extract_images_sharded(li, lk_), steps, max(warmup, 8))
        assert sum(len(v[1]) for v in out.values()) == m_local
        return {"value": m_total / s, "unit": UNITS["cfg3"], "ms_per_step": s * 1e3,
                "h2d_bytes_per_step": int(sum(a.nbytes for a in host_imgs) + m_local * 32),
                "d2h_bytes_per_step": int(m_local * 64),
                "api": f"sharded.extract_images_sharded -> describe_batch({tag} images, keypoints (N,4)), {memory} host arrays"}

    e2e_u8 = e2e_leg([cx.pinned(a) for a in imgs], "u8", "page-locked")
    e2e = e2e_leg([a.astype(np.float64) for a in imgs], "f64", "ordinary (pageable) numpy")
    hbm = sum(a.nbytes for a in imgs) + m_local * (32 + 64)
    rec = {
        "workload": W.DESCRIPTIONS["cfg3"], "value": m_total / sec, "unit": UNITS["cfg3"], "ms_per_step": sec * 1e3,
        "steps": steps, "warmup": warmup, "scaling": "strong", "images": count, "images_this_rank": len(mine),
        "descriptors": m_total, "e2e": e2e, "e2e_u8": e2e_u8, "gpu_launches": int(launches),
        "roofline": cx.extract_roofline(m_local, sec, clocks_out.get("sm_mhz") or 1965.0, hbm),
        "timing": "CUDA events around this rank's images (resident in HBM, 0.7 GB cycled per pass > L2), max over ranks",
    }
    if cpu and cx.rank == 0 and cx.world == 1:
        import oracle
        rec["cpu_baseline"] = cpu_sample("cfg3", oracle.cpu_threads())
    return rec


def run_cfg4(cx: Ctx, steps: int, warmup: int, cpu: bool, clocks_out: dict):
    """1 M x 1 M top-2 + ratio test: train set broadcast from rank 0 (NCCL), queries sharded, triples gathered."""
    torch, eng = cx.torch, cx.eng
    from paper_1609_03986_b200 import sharded
    W = wl()
    q, t, (dup_q, _) = W.cfg4_sets()
    nq, nt = len(q), len(t)
    b, e = sharded.shard_bounds(nq, cx.world)[cx.rank]
    d_q = torch.from_numpy(q[b:e]).to(cx.dev)
    d_t = torch.from_numpy(t).to(cx.dev) if cx.rank == 0 else torch.empty(t.shape, dtype=torch.uint8, device=cx.dev)
    res = {}

    def step(ev):
        if ev: ev[0].record()
        res["r"] = sharded.match_top2_sharded_device(d_q, d_t, nq)
        if ev: ev[1].record()

    launches0 = eng.launch_count
    with ClockSampler(cx.local) as clocks:
        (t_dev,), _ = cx.time_events(step, steps, warmup)
    launches = (eng.launch_count - launches0) * steps // (steps + warmup)
    clocks_out.update(clocks.summary())
    sec = t_dev / steps
    r = res["r"].cpu().numpy()
    planted_found = int((r[1][dup_q] == 0).sum())
    del d_q, d_t, res

    hq, ht = cx.pinned(q), cx.pinned(t)
    s_e2e, rows = cx.time_wall(lambda: sharded.match_sharded_host(hq, ht, ratio=W.RATIO), steps, warmup)
    rec = {
        "workload": W.DESCRIPTIONS["cfg4"], "value": nq * nt / sec, "unit": UNITS["cfg4"], "ms_per_step": sec * 1e3,
        "steps": steps, "warmup": warmup, "scaling": "strong", "queries": nq, "train": nt,
        "queries_this_rank": e - b, "planted_copies_found": planted_found, "planted_copies": int(len(dup_q)),
        "ratio_matches": int(len(rows)),
        "e2e": {"value": nq * nt / s_e2e, "unit": UNITS["cfg4"], "ms_per_step": s_e2e * 1e3,
                "h2d_bytes_per_step": int((e - b) * 64 + (nt * 64 if cx.rank == 0 else 0)),
                "d2h_bytes_per_step": int(12 * nq),
                "api": "sharded.match_sharded_host(queries, train, ratio=0.8): page-locked host arrays in, (M,4) int32 rows out"},
        "gpu_launches": int(launches),
        "roofline": cx.match_roofline((e - b) * nt, sec, clocks_out.get("sm_mhz") or 1965.0, (e - b) * 64 + nt * 64 + 12 * (e - b),
                                      "bit->int8 expansion of both sets, GEMM + top-2 epilogue, split merge"
                                      + ("; NCCL broadcast + all_gather" if cx.world > 1 else "")),
        "timing": "CUDA events on the launching stream around expand + match (+ NCCL broadcast / gather at N > 1), max over "
                  "ranks; operands (2 x 64 MB packed, 2 x 512 MB expanded) exceed L2 and L2 is flushed between steps",
    }
    if cpu and cx.rank == 0 and cx.world == 1:
        import oracle
        rec["cpu_baseline"] = cpu_sample("cfg4", oracle.cpu_threads())
    return rec


def run_cfg5(cx: Ctx, steps: int, warmup: int, cpu: bool, clocks_out: dict):
    """256 images x 8 000 keypoints: extraction sharded by image, one all-gather of the descriptor sets,
    all 32 640 (i < j) pairs dealt round-robin, each matched with ratio 0.8 + cross-check."""
    torch, eng = cx.torch, cx.eng
    from paper_1609_03986_b200 import sharded
    W = wl()
    w, h, n, _, _, count = W.IMAGE_CONFIGS["cfg5"]
    mine = list(range(cx.rank, count, cx.world))
    imgs, kps = W.images_and_keypoints("cfg5", mine)
    pairs_total = count * (count - 1) // 2
    full = [None] * count

    def whole_job(host_imgs):
        li, lk_ = list(full), list(full)
        for i, a, k in zip(mine, host_imgs, kps):
            li[i], lk_[i] = a, k
        local = sharded.extract_images_sharded(li, lk_)
        sets = sharded.all_gather_descriptor_sets({i: v[1] for i, v in local.items()}, count, device=cx.dev)
        return sets, sharded.match_all_pairs_resident(sets, ratio=W.RATIO, cross_check=True, num_images=count)

    # device-resident leg: descriptor sets already in HBM as resident sets; the step = this rank's pairs
    sets, _ = whole_job(imgs)
    rows_per_set = [int(s.shape[0]) for s in sets]
    resident = sharded.create_resident_sets(sets, count)
    my_pairs = sharded.pairs_for_rank(count, cx.rank, cx.world)
    compares_local = sum(2 * rows_per_set[i] * rows_per_set[j] for i, j in my_pairs)
    compares_total = cx.sum_over_ranks(compares_local)[0]
    launches0 = eng.launch_count
    with ClockSampler(cx.local) as clocks:
        sec, out = cx.time_wall(lambda: sharded.match_all_pairs_resident(sets, ratio=W.RATIO, cross_check=True,
                                                                         num_images=count, resident=resident),
                                steps, warmup)
    launches = (eng.launch_count - launches0) * steps // (steps + warmup)
    clocks_out.update(clocks.summary())
    kept_rows = int(cx.sum_over_ranks(sum(len(v) for v in out.values()))[0])
    for s in resident.values():
        s.close()
    del resident, sets, out

    def e2e_leg(host_imgs, tag, memory):
        s, o = cx.time_wall(lambda: whole_job(host_imgs)[1], steps, max(warmup, 8))
        return {"value": pairs_total / s, "unit": UNITS["cfg5"], "ms_per_step": s * 1e3,
                "compares_per_s": compares_total / s,
                "h2d_bytes_per_step": int(sum(a.nbytes for a in host_imgs) + sum(rows_per_set[i] for i in mine) * 32),
                "d2h_bytes_per_step": int(sum(rows_per_set[i] for i in mine) * 64 + 16 * sum(len(v) for v in o.values())),
                "api": f"extract_images_sharded({tag} images, {memory}) -> all_gather_descriptor_sets -> "
                       "match_all_pairs_resident(ratio=0.8, cross_check=True): host images in, per-pair (M,4) rows out"}

    e2e_u8 = e2e_leg([cx.pinned(a) for a in imgs], "u8", "page-locked")
    e2e = e2e_leg([a.astype(np.float64) for a in imgs], "f64", "ordinary numpy")
    rec = {
        "workload": W.DESCRIPTIONS["cfg5"], "value": pairs_total / sec, "unit": UNITS["cfg5"], "ms_per_step": sec * 1e3,
        "steps": steps, "warmup": warmup, "scaling": "strong", "images": count, "pairs": pairs_total,
        "pairs_this_rank": len(my_pairs), "compares_per_s": compares_total / sec, "matches_kept": kept_rows,
        "e2e": e2e, "e2e_u8": e2e_u8, "gpu_launches": int(launches),
        "roofline": cx.match_roofline(compares_local, sec, clocks_out.get("sm_mhz") or 1965.0,
                                      sum(rows_per_set) * 64 + 16 * kept_rows,
                                      "forward + reverse GEMMs of every pair over resident expanded sets, the on-device "
                                      "filter pass, and the D2H of the surviving rows"),
        "timing": "host clock around match_all_pairs_resident over resident sets (a synchronous call: launches, filter, "
                  "result D2H), device synchronised on both sides, max over ranks; 0.27 GB of expanded operands cycle "
                  "through L2 per pass and L2 is flushed between steps",
    }
    if cpu and cx.rank == 0 and cx.world == 1:
        import oracle
        rec["cpu_baseline"] = cpu_sample("cfg5", oracle.cpu_threads())
    return rec


def run_ours(args):
    cx = Ctx(args)
    runners = {"cfg1": lambda *a: run_image_step(cx, "cfg1", *a), "cfg2": lambda *a: run_image_step(cx, "cfg2", *a),
               "cfg3": lambda *a: run_cfg3(cx, *a), "cfg4": lambda *a: run_cfg4(cx, *a), "cfg5": lambda *a: run_cfg5(cx, *a)}
    head = "cfg2" if args.workload == "all" else args.workload
    cpu = not args.no_cpu_baseline
    clocks = {}
    rec = runners[head](args.steps, args.warmup, cpu, clocks)
    configs = {}
    if args.workload == "all":
        side_steps, side_warm = min(args.steps, 3), 3
        for cfg in ("cfg1", "cfg3", "cfg4", "cfg5"):
            if cfg in args.skip:
                continue
            t0 = time.perf_counter()
            c = {}
            sub = runners[cfg](min(args.steps, 20) if cfg == "cfg1" else side_steps, side_warm, cpu, c)
            sub["clocks"] = c
            sub["bench_wall_s"] = time.perf_counter() - t0
            configs[cfg] = sub
            print(f"[bench] {cfg}: {sub['value']:.4g} {sub['unit'].split(' (')[0]} "
                  f"(e2e {sub['e2e']['value']:.4g}) in {sub['bench_wall_s']:.1f} s", file=sys.stderr, flush=True)
        configs["cfg2"] = {k: rec[k] for k in ("workload", "value", "unit", "ms_per_step", "scaling", "descriptors_per_s",
                                               "compares_per_s") if k in rec}
        configs["cfg2"]["e2e"] = rec["e2e"]
    if cx.rank == 0:
        line = {
            "metric": METRICS[head], "value": rec["value"], "unit": rec["unit"], "n_gpus": cx.world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": rec["ms_per_step"], "higher_is_better": True, "scaling": rec["scaling"],
            "vs_baseline": None,
            "dtype": (("fp32 resampling into 16-bit planes + fp32 estimate under a proven bound, exact f64 recompute of every "
                       "undecided bit" if cx.ev >= 5 else
                       "f64 resampling, " + ("fp32 estimate + exact f64 recompute" if cx.ev >= 2 else "f64 SSD")) +
                      " (extraction) / " + ({3: "int8 tcgen05, int32 accumulate", 4: "e2m1 tcgen05 (mxf4, unit scales), f32 accumulate"}.get(cx.mv, "u32 xor+popc")) +
                      " (matching); results bit-exact"),
            "data": "synthetic",
            "config": {"workload": rec["workload"], "phase": args.phase, "timing": rec["timing"],
                       "l2": "256 MiB device memset between steps, outside the timed spans; the sharded configurations' "
                             "inputs also exceed L2"},
            "clocks": clocks, "e2e": rec["e2e"], "gpu_launches": rec["gpu_launches"], "roofline": rec["roofline"],
            "cpu_baseline": rec.get("cpu_baseline"), "device": cx.eng.name, "sm_count": cx.eng.sm_count,
        }
        for k, v in rec.items():
            if k not in line and k not in ("workload", "timing", "steps", "warmup"):
                line[k] = v
        if configs:
            line["configs"] = dict(sorted(configs.items()))
        emit(line)
    if cx.use_dist:
        cx.dist.destroy_process_group()


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
    ap.add_argument("--workload", choices=["all", "cfg1", "cfg2", "cfg3", "cfg4", "cfg5"], default="all")
    ap.add_argument("--skip", default="", help="comma list of side configurations to leave out of --workload all")
    ap.add_argument("--phase", choices=["both", "extract", "match"], default="both")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--match-variant", type=int, default=None, help="override the matcher kernel variant (0..4)")
    ap.add_argument("--extract-variant", type=int, default=None, help="override the extraction kernel variant (0..4)")
    args = ap.parse_args()
    args.skip = set(filter(None, args.skip.split(",")))
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
