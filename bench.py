#!/usr/bin/env python3
"""Benchmark of the bitsliced 3DES-EDE ECB hot path (arXiv 2007.10752) on B200.

Workload (BASELINE.json configs[1], top of the paper-style size sweep): 3DES-EDE
ECB **encrypt** of 2^27 blocks = 1 GiB of synthetic plaintext per GPU, 3-key
(NIST SP 800-67 sample keys).  One step = one pass of the whole hot path (one
fused kernel launch: load, transpose, 48 rounds, transpose, store) over the
1 GiB batch.  Inputs (1 GiB) and outputs (1 GiB) exceed the 126 MB L2, so no
flush is needed between steps.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 runs under torchrun, one process per GPU, each rank encrypting its own
1 GiB block-range shard of the global data (weak scaling, no collective on the
data path; NCCL only for the barrier and the max-over-ranks time).

``--impl reference`` times the CPU oracle (oracle/, the literal char-per-bit
C implementation, OpenMP over blocks as in the paper's CPU baseline)
on a bounded sample of the same workload; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synthetic  # noqa: E402

METRIC = "3DES-ECB encrypt GB/s per B200 and at 1/2/4/8 GPUs; % of INT32/LOP3 roofline"
UNIT = "GB/s"
BLOCKS_PER_GPU = 1 << 27          # 1 GiB per GPU
WORKLOAD = "3DES-EDE ECB encrypt, 1 GiB (2^27 blocks) per GPU, 3-key (SP 800-67 sample keys), synthetic splitmix64 plaintext"
SM_COUNT_NOMINAL = 148
LOP3_LANES_PER_SM = 64            # B300_MICROARCH.md: LOP3 on the alu pipe, rt_SMSP = 2 -> 16 lanes/clk/SMSP
HBM_PEAK_FALLBACK = 6650.0        # B200_PROFILING.md fallback (GB/s)
E2E_MAX_BLOCKS = 1 << 27          # e2e leg: at most 1 GiB of pinned host memory per direction

# --workload: c2 (default) is the driver's bench line; c4 and c5 are SURVEY §8d's
# multi-GPU rows, runnable at any N (block-range shards of a fixed total).
WORKLOADS = {
    "c2": {"per_gpu": BLOCKS_PER_GPU, "total": None, "roundtrip": False, "scaling": "weak",
           "desc": WORKLOAD},
    "c4": {"per_gpu": None, "total": 1 << 30, "roundtrip": False, "scaling": "strong",
           "desc": "3DES-EDE ECB encrypt, 8 GiB (2^30 blocks) in total, block-range shards over the GPUs, "
                   "3-key (SP 800-67 sample keys), synthetic splitmix64 plaintext (BASELINE.json configs[3])"},
    "c5": {"per_gpu": None, "total": 1 << 33, "roundtrip": True, "scaling": "strong",
           "desc": "3DES-EDE ECB encrypt-then-decrypt round trip, 64 GiB (2^33 blocks) in total, block-range "
                   "shards over the GPUs, 3-key, synthetic splitmix64 plaintext (BASELINE.json configs[4]); "
                   "value = plaintext bytes round-tripped per second"},
}


def env_int(name, default):
    try:
        return int(os.environ.get(name, default))
    except ValueError:
        return default


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except (OSError, ValueError):
        return {"hbm_gbs": HBM_PEAK_FALLBACK, "sm_max_mhz": 1965.0}, "fallback"


def read_traffic():
    """Per-block DRAM bytes of the kernel from the committed ncu capture, if any."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["dram_bytes_per_block"]), d.get("source", path)
    except (OSError, ValueError, KeyError):
        return None, None


class ClockSampler:
    """Samples SM clock and throttle reasons via NVML every ~10 ms while running."""

    def __init__(self, pci_bus_id, fallback_index):
        self.samples, self.reasons, self.ok = [], set(), False
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = None
            for bus in ([pci_bus_id, "0000" + pci_bus_id] if pci_bus_id else []):
                try:
                    self.h = pynvml.nvmlDeviceGetHandleByPciBusId(bus)
                    break
                except Exception:
                    pass
            if self.h is None:
                self.h = pynvml.nvmlDeviceGetHandleByIndex(fallback_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.ok = False
        self.names = {}
        if self.ok:
            for attr, name in [("nvmlClocksEventReasonGpuIdle", "gpu_idle"),
                               ("nvmlClocksEventReasonApplicationsClocksSetting", "applications_clocks_setting"),
                               ("nvmlClocksEventReasonSwPowerCap", "sw_power_cap"),
                               ("nvmlClocksEventReasonHwSlowdown", "hw_slowdown"),
                               ("nvmlClocksEventReasonSyncBoost", "sync_boost"),
                               ("nvmlClocksEventReasonSwThermalSlowdown", "sw_thermal_slowdown"),
                               ("nvmlClocksEventReasonHwThermalSlowdown", "hw_thermal_slowdown"),
                               ("nvmlClocksEventReasonHwPowerBrakeSlowdown", "hw_power_brake_slowdown")]:
                v = getattr(self.nv, attr, None)
                if v is None:
                    v = getattr(self.nv, attr.replace("ClocksEvent", "ClocksThrottle"), None)
                if v is not None:
                    self.names[v] = name

    def _run(self):
        nv = self.nv
        get_reasons = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
            nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = get_reasons(self.h)
                for bit, name in self.names.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["nvml_unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "sm_mhz_min": min(self.samples), "samples": len(self.samples),
                "reasons": sorted(self.reasons)}


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def oracle_rate(budget_s: float, max_blocks: int):
    """Time the oracle (as it stands) on a bounded sample of the workload.

    Returns (GB/s, threads used, sample description, seconds)."""
    import oracle
    keys = synthetic.KEYS_3KEY
    dt, probe = 0.0, 1 << 12
    while probe < max_blocks:          # probe until the sample takes >= 0.5 s (threads warm)
        p = synthetic.plaintext_bytes(0, probe)
        out = np.empty_like(p)
        t0 = time.perf_counter()
        oracle.tdes_ecb_into(*keys, p, out)
        dt = max(time.perf_counter() - t0, 1e-6)
        if dt >= 0.5:
            break
        probe *= 4
    n = int(min(max_blocks, max(probe, budget_s * probe / dt)))
    n -= n % 1024
    p = synthetic.plaintext_bytes(0, n)
    out = np.empty_like(p)
    t0 = time.perf_counter()
    used = oracle.tdes_ecb_into(*keys, p, out)
    dt = time.perf_counter() - t0
    return n * 8 / dt / 1e9, used, f"first {n} blocks ({n * 8 / 2**20:.1f} MiB) of the workload, wall clock, OpenMP over blocks", dt


# ------------------------------------------------------------ reference arm --

def run_reference(args, rank, world):
    if rank != 0:
        return 0
    import oracle
    keys = synthetic.KEYS_3KEY
    # size each step so the whole --steps K --warmup W run ends within ~2 minutes
    probe = 1 << 12
    p = synthetic.plaintext_bytes(0, probe)
    out = np.empty_like(p)
    t0 = time.perf_counter()
    oracle.tdes_ecb_into(*keys, p, out)
    dt = max(time.perf_counter() - t0, 1e-6)
    per_step_s = min(10.0, 120.0 / max(1, args.steps + args.warmup))
    n = int(max(1024, min(BLOCKS_PER_GPU, per_step_s * probe / dt)))
    n -= n % 1024
    p = synthetic.plaintext_bytes(0, n)
    out = np.empty_like(p)
    used = 1
    for _ in range(args.warmup):
        used = oracle.tdes_ecb_into(*keys, p, out)
    ts = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        used = oracle.tdes_ecb_into(*keys, p, out)
        ts.append(time.perf_counter() - t0)
    total = sum(ts)
    value = args.steps * n * 8 / total / 1e9
    sample = f"first {n} blocks ({n * 8 / 2**20:.2f} MiB) of the 1 GiB workload per step, wall clock"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u8",
        "data": "synthetic",
        "config": {"workload": WORKLOAD + " (oracle timed on a bounded sample)", "blocks_per_step": n,
                   "parallelism": "OpenMP over blocks on host cores (PAPER.md:140)"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": used, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    emit(line)
    return 0


# ----------------------------------------------------------------- our arm --

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_2007_10752_b200 as tdes

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    distributed = world > 1 or "TORCHELASTIC_RUN_ID" in os.environ  # torchrun: exercise NCCL even at N=1
    if distributed:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if distributed:
            dist.barrier()

    from paper_2007_10752_b200 import shard
    wl = WORKLOADS[args.workload]
    total_blocks = wl["total"] if wl["total"] is not None else wl["per_gpu"] * world
    lo, hi = shard.shard_range(total_blocks, world, rank)
    n = hi - lo
    free_b, _ = torch.cuda.mem_get_info(dev)
    if 16 * n + (1 << 30) > free_b:
        raise SystemExit(f"workload {args.workload}: {16 * n / 2**30:.0f} GiB of buffers per GPU "
                         f"do not fit in {free_b / 2**30:.0f} GiB free; use more GPUs")
    launches_per_step = 2 if wl["roundtrip"] else 1
    sched = tdes.key_schedule(*synthetic.KEYS_3KEY)
    x = torch.empty(8 * n, dtype=torch.uint8, device=dev)
    y = torch.empty_like(x)
    tdes.fill_splitmix64(x, first_index=lo)
    stream = torch.cuda.current_stream(dev)
    handle = stream.cuda_stream

    # ---- LOP3 peak microbenchmark (roofline cross-check, same process) ----
    sms, occ = tdes.device_geometry()
    sink = torch.empty(sms * 8 * 256, dtype=torch.int32, device=dev)
    tdes.lop3_peak_launch(sink, sms * 8, 256, 1024)
    torch.cuda.synchronize()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    ops = tdes.lop3_peak_launch(sink, sms * 8, 256, 8192)
    ev1.record(stream)
    ev1.synchronize()
    lop3_peak_meas = ops / (ev0.elapsed_time(ev1) * 1e-3) / 1e12   # Tops/s

    def step_launches():
        """One step: one fused launch (c2, c4) or encrypt + in-place decrypt (c5)."""
        yield lambda: tdes.ecb_encrypt_ptr(sched, x.data_ptr(), y.data_ptr(), n, handle)
        if wl["roundtrip"]:
            yield lambda: tdes.ecb_decrypt_ptr(sched, y.data_ptr(), y.data_ptr(), n, handle)

    # ---- warmup ----
    for _ in range(args.warmup):
        for launch in step_launches():
            launch()
    torch.cuda.synchronize()

    # ---- timed region: K steps ----
    nl = args.steps * launches_per_step
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(nl)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(nl)]
    t_begin, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    props = torch.cuda.get_device_properties(dev)
    bus = None
    if hasattr(props, "pci_bus_id"):
        bus = f"{getattr(props, 'pci_domain_id', 0):04x}:{props.pci_bus_id:02x}:{getattr(props, 'pci_device_id', 0):02x}.0"
    sampler = ClockSampler(bus, local_rank)
    barrier()
    torch.cuda.synchronize()
    with sampler:
        t_begin.record(stream)
        k = 0
        for _ in range(args.steps):
            for launch in step_launches():
                starts[k].record(stream)
                launch()
                ends[k].record(stream)
                k += 1
        t_end.record(stream)
        torch.cuda.synchronize()
    barrier()
    elapsed_ms = t_begin.elapsed_time(t_end)
    kern_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    elapsed_ms = shard.max_over_ranks(elapsed_ms)
    clocks = sampler.summary()

    # ---- device-side sanity: decrypt restores the plaintext; digest ----
    if wl["roundtrip"]:
        mismatch = tdes.count_mismatch(y, x)       # y = dec(enc(x)) after the last step
        tdes.ecb_encrypt_ptr(sched, x.data_ptr(), y.data_ptr(), n, handle)
        digest = tdes.sum64(y)
    else:
        digest = tdes.sum64(y)
        tdes.ecb_decrypt_ptr(sched, y.data_ptr(), y.data_ptr(), n, handle)
        mismatch = tdes.count_mismatch(y, x)
    mismatch = shard.sum_over_ranks(mismatch)
    digest = shard.sum_u64_over_ranks(digest)

    # ---- e2e: same metric through the host-buffer C-ABI call ----
    # (a bounded prefix of the shard for c4/c5: at most 1 GiB of pinned host memory per direction)
    ne = min(n, E2E_MAX_BLOCKS)
    del y
    torch.cuda.empty_cache()
    hin = torch.empty(8 * ne, dtype=torch.uint8).pin_memory()
    hin.copy_(x[:8 * ne].cpu())
    del x
    torch.cuda.empty_cache()
    hout = torch.empty_like(hin).pin_memory()
    pipe = tdes.HostPipeline(chunk_blocks=1 << 22, nstreams=3, device=dev)  # tools/e2e_sweep.py
    e2e_steps = max(1, min(args.steps, 10))
    pipe.run(sched, hin, hout)      # warmup
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(e2e_steps):
        pipe.run(sched, hin, hout)
        if wl["roundtrip"]:
            pipe.run(sched, hout, hout, decrypt=True)
        for s in pipe.streams:
            stream.wait_stream(s)
    e1.record(stream)
    e1.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    e2e_ms = shard.max_over_ranks(e2e_ms)
    e2e_value = e2e_steps * ne * world * 8 / (e2e_ms * 1e-3) / 1e9

    if rank == 0:
        peaks, peaks_src = read_peaks()
        info = tdes.kernel_info()
        T = info.sbox_lop3_total
        # Algorithmic ALU-pipe ops per block: per round T S-box gates +
        # 32 Feistel XORs, per 32 blocks.  The 48 key XORs per round run on the FMA
        # pipe (IMAD), so they are reported beside the headline, not inside it.
        g_alg = 48 * (T + 32) / 32
        g_alg_kx = 48 * (48 + T + 32) / 32           # SURVEY §8d G_alg, key XORs included
        avg_kern_s = sum(kern_ms) / len(kern_ms) * 1e-3
        achieved = g_alg * n / avg_kern_s / 1e12    # Tops/s on this rank's launches
        sm_max = float(peaks.get("sm_max_mhz", 1965.0))
        peak = sms * LOP3_LANES_PER_SM * sm_max * 1e6 / 1e12
        tb, tsrc = read_traffic()
        value = args.steps * total_blocks * 8 / (elapsed_ms * 1e-3) / 1e9
        hbm_gbs = 16 * n / avg_kern_s / 1e9
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": elapsed_ms / args.steps, "higher_is_better": True,
            "scaling": wl["scaling"], "vs_baseline": None, "dtype": "u32", "data": "synthetic",
            "config": {"workload": wl["desc"], "name": args.workload, "blocks_per_gpu": n,
                       "bytes_per_gpu": n * 8, "total_blocks": total_blocks,
                       "op": "encrypt+decrypt" if wl["roundtrip"] else "encrypt", "keys": "3-key",
                       "parallelism": f"dp{world} (block-range shards)",
                       "l2": f"inputs and outputs {n * 8 / 2**30:.2f} GiB per GPU > 126 MB L2; no flush needed",
                       "Gblocks_per_s": value / 8},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "Tops/s",
                         "frac": achieved / peak,
                         "traffic": (tb * n if tb is not None else None),
                         "ops_per_block": g_alg, "sbox_lop3_total": T,
                         "ops_per_block_incl_key_xor": g_alg_kx,
                         "frac_incl_key_xor": g_alg_kx * n / avg_kern_s / 1e12 / peak,
                         "peak_basis": f"{sms} SMs x {LOP3_LANES_PER_SM} LOP3 lanes/clk x {sm_max:.0f} MHz (sm_max_mhz, {peaks_src})",
                         "peak_microbench": lop3_peak_meas,
                         "frac_of_microbench": achieved / lop3_peak_meas,
                         "kernel_ms_avg": avg_kern_s * 1e3,
                         "kernel_ms_p10_p50_p90": [round(float(np.percentile(kern_ms, q)), 5) for q in (10, 50, 90)],
                         "hbm": {"achieved_gbs": hbm_gbs, "peak_gbs": float(peaks.get("hbm_gbs", HBM_PEAK_FALLBACK)),
                                 "frac": hbm_gbs / float(peaks.get("hbm_gbs", HBM_PEAK_FALLBACK)),
                                 "bytes_per_block": 16, "peak_source": peaks_src},
                         "traffic_source": tsrc},
            "clocks": clocks,
            "e2e": {"value": e2e_value, "unit": UNIT,
                    "h2d_bytes_per_step": 8 * ne * launches_per_step,
                    "d2h_bytes_per_step": 8 * ne * launches_per_step,
                    "how": "tdes_ecb_crypt_host: pinned host in/out, 32 MiB chunks on 3 streams (H2D, kernel, D2H overlapped)"
                           + ("" if ne == n else f"; first {ne} blocks of each shard")
                           + ("; encrypt then decrypt in place" if wl["roundtrip"] else ""),
                    "steps": e2e_steps},
            "gpu_launches": nl,
            "check": {"device_roundtrip_mismatch_blocks": mismatch, "ciphertext_sum64": f"{digest:016x}"},
        }
        if world == 1 and not args.no_cpu_baseline and args.workload == "c2":
            v, used, sample, secs = oracle_rate(args.cpu_seconds, BLOCKS_PER_GPU)
            line["cpu_baseline"] = {"value": v, "unit": UNIT, "cores": used, "kind": "oracle",
                                    "sample": sample, "seconds": secs, "host_cores": host_cores()}
        emit(line)
    if distributed:
        dist.barrier()
        dist.destroy_process_group()
    return 0


def _json_stdout():
    """Keep fd 1 for the one JSON line: libraries that print banners to stdout
    from C (NCCL's version line at communicator init) are routed to stderr."""
    out = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    return out


def emit(line: dict):
    print(json.dumps(line), file=JSON_OUT, flush=True)


JSON_OUT = sys.stdout


def main():
    global JSON_OUT
    JSON_OUT = _json_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS),
                    help="c2: 1 GiB encrypt per GPU (default, weak scaling); c4: 8 GiB total encrypt; "
                         "c5: 64 GiB total encrypt+decrypt round trip (strong scaling)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    rank = env_int("RANK", 0)
    world = env_int("WORLD_SIZE", 1)
    local_rank = env_int("LOCAL_RANK", 0)
    if args.impl == "reference":
        return run_reference(args, rank, world)
    return run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    sys.exit(main())
