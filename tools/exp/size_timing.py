"""Per-size launch timing of the 3DES path, three ways (dev aid; prints a table).

  idle   events around one launch on an idle GPU: device time + host submission
         latency (what round 1's C2 sweep reported)
  queued one launch queued behind a ~0.3 ms device-side sleep, so the host has
         submitted it before the first event fires: device time of the launch
         alone (front-end + kernel), no host latency
  b2b    20 launches back to back / 20

  python tools/exp/size_timing.py [--modes 0,1,2] [--lo 17] [--hi 27]
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402


def median(v):
    v = sorted(v)
    return v[len(v) // 2]


def timings(fn, reps=15):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    idle, queued = [], []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        idle.append(a.elapsed_time(b))
        torch.cuda._sleep(600_000)          # ~0.3 ms at 1.9 GHz
        a.record()
        fn()
        b.record()
        b.synchronize()
        queued.append(a.elapsed_time(b))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(600_000)
    a.record()
    for _ in range(20):
        fn()
    b.record()
    b.synchronize()
    return median(idle), median(queued), a.elapsed_time(b) / 20


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--modes", default="0")
    ap.add_argument("--lo", type=int, default=17)
    ap.add_argument("--hi", type=int, default=27)
    ap.add_argument("--decrypt", action="store_true")
    a = ap.parse_args()
    s = tdes.key_schedule(*synthetic.KEYS_3KEY)
    N = 1 << a.hi
    x = torch.empty(8 * N, dtype=torch.uint8, device="cuda")
    tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    modes = [int(m) for m in a.modes.split(",")]
    print("log2n mode   idle_us queued_us  b2b_us | idle_GBs queued_GBs b2b_GBs", flush=True)
    for e in range(a.lo, a.hi + 1):
        n = 1 << e
        xs, ys = x[:8 * n], y[:8 * n]
        for m in modes:
            r = timings(lambda: tdes.ecb_crypt_mode(xs, s, m, decrypt=a.decrypt, out=ys))
            print(f"{e:5d} {m:4d} " + " ".join(f"{v * 1e3:9.1f}" for v in r) + " | "
                  + " ".join(f"{n * 8 / v / 1e6:9.1f}" for v in r), flush=True)


if __name__ == "__main__":
    main()
