"""TEST INFRASTRUCTURE (calls oracle/). BASELINE.json config 2: paper-style size sweep 1 MiB .. 1 GiB, 3DES-ECB encrypt and
decrypt on one B200, with the CPU oracle timed beside it on the host cores.  Writes a
markdown table (default profiles/sweep_c2.md).

Per size: device time of one launch (median of 10, CUDA events, data resident), GB/s;
bit-exactness vs the oracle (every block up to 2^20 blocks, 4096 sampled blocks plus
the first/last 1024 above that) for both directions; the oracle's wall time on the
host cores (full size while the estimate stays under the cap, else a timed sample
scaled up, marked "~").  Config 3 (1-key and 2-key on 256 MiB) rides along.
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the timed CPU baseline)
import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402


def dev_time(fn, reps=10):
    """(queued, idle, back-to-back) ms per launch, medians of `reps`.

    queued: the launch is submitted behind a ~0.3 ms device-side sleep, so the
            events bracket the launch's device time alone (front end + kernel);
    idle:   events around one launch on an idle GPU (adds host submission latency);
    b2b:    20 launches back to back, per launch."""
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    q, i = [], []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        i.append(a.elapsed_time(b))
        torch.cuda._sleep(600_000)
        a.record()
        fn()
        b.record()
        b.synchronize()
        q.append(a.elapsed_time(b))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(600_000)
    a.record()
    for _ in range(20):
        fn()
    b.record()
    b.synchronize()
    return sorted(q)[len(q) // 2], sorted(i)[len(i) // 2], a.elapsed_time(b) / 20


def check(keys, x, y, decrypt, n):
    if n <= 1 << 20:
        exp = oracle.tdes_ecb(*keys, synthetic.plaintext_bytes(0, n), decrypt=decrypt)
        return np.array_equal(y.cpu().numpy(), exp), n
    rng = np.random.default_rng(n + decrypt)
    idx = np.unique(np.concatenate([rng.integers(0, n, 4096), np.arange(1024), np.arange(n - 1024, n)]))
    got = y.view(-1, 8)[torch.from_numpy(idx).cuda()].cpu().numpy().reshape(-1)
    exp = oracle.tdes_ecb(*keys, synthetic.gather_blocks(idx), decrypt=decrypt)
    return np.array_equal(got, exp), len(idx)


def oracle_time(keys, n, cap_s, rate, threads=0):
    """Full-size oracle wall time if it fits the cap, else a timed sample scaled up
    (threads <= 0: all OpenMP threads; SURVEY 8(d) asks for 1 thread and all)."""
    est = n / rate if rate else 0
    m = n if est <= cap_s else max(1 << 14, int(cap_s * rate) // 4)
    p = synthetic.plaintext_bytes(0, m)
    out = np.empty_like(p)
    t0 = time.perf_counter()
    oracle.tdes_ecb_into(*keys, p, out, threads=threads)
    dt = time.perf_counter() - t0
    return dt * n / m, m == n, m / dt


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="profiles/sweep_c2.md")
    ap.add_argument("--cap", type=float, default=20.0, help="oracle seconds per point")
    a = ap.parse_args()
    N = 1 << 27
    x = torch.empty(8 * N, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    cores = len(os.sched_getaffinity(0))
    rate = rate1 = None
    lines = ["# Config 2: size sweep, 3DES-EDE ECB on one B200 vs the oracle on host cores", "",
             f"GPU: {torch.cuda.get_device_name(0)}; host cores used by the oracle: {cores} (OpenMP over blocks).",
             "Device time = one launch queued behind a device-side sleep (median of 10, CUDA events, data",
             "resident in HBM): the launch's own device time, no host submission latency.  Beside it: the",
             "same launch on an idle GPU (adds the host's submission latency) and 20 launches back to back.",
             "Oracle = `oracle/tdes_oracle.c` (char per bit, as in the paper), wall clock;",
             "`~` = extrapolated from a timed sample (the full size would exceed the per-point cap).",
             "The oracle is timed on all host threads and on 1 thread (SURVEY 8(d)).", "",
             "| blocks | bytes | op | keys | GPU ms | GPU GB/s | idle-launch GB/s | back-to-back GB/s | bit-exact (blocks checked) | oracle s | oracle GB/s | GPU/oracle | oracle 1-thread s | GPU/oracle 1-thread |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    points = [(e, op, "3-key") for e in range(17, 28) for op in ("enc", "dec")]
    points += [(25, op, k) for k in ("1-key", "2-key") for op in ("enc", "dec")]
    keysets = {"3-key": synthetic.KEYS_3KEY, "2-key": synthetic.KEYS_2KEY, "1-key": synthetic.KEYS_1KEY}
    for e, op, kname in points:
        n = 1 << e
        keys = keysets[kname]
        s = tdes.key_schedule(*keys)
        dec = op == "dec"
        fn = tdes.ecb_decrypt if dec else tdes.ecb_encrypt
        xs, ys = x[:8 * n], y[:8 * n]
        ms, ms_idle, ms_b2b = dev_time(lambda: fn(xs, s, out=ys))
        ok, nchk = check(keys, xs, ys, dec, n)
        osec, full, r = oracle_time(keys, n, a.cap, rate)
        rate = rate or r
        osec1, full1, r1 = oracle_time(keys, n, a.cap / 4, rate1, threads=1)
        rate1 = rate1 or r1
        gbs = n * 8 / ms / 1e6
        ogbs = n * 8 / osec / 1e9
        lines.append(f"| 2^{e} | {n * 8 / 2**20:g} MiB | {op} | {kname} | {ms:.4f} | {gbs:.1f} | "
                     f"{n * 8 / ms_idle / 1e6:.1f} | {n * 8 / ms_b2b / 1e6:.1f} | "
                     f"{'yes' if ok else 'NO'} ({nchk}) | {'' if full else '~'}{osec:.2f} | {ogbs:.4f} | "
                     f"{gbs / ogbs:.0f}x | {'' if full1 else '~'}{osec1:.2f} | {gbs / (n * 8 / osec1 / 1e9):.0f}x |")
        print(lines[-1], flush=True)
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()
