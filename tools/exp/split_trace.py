"""Per-round clock64 timeline of the split kernel (experiment aid).

  python tools/exp/split_trace_build.py   # -> tools/exp/strace.so
  TDES_LIB_PATH=tools/exp/strace.so python tools/exp/split_trace.py [nblocks ...]
"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402

s = tdes.key_schedule(*synthetic.KEYS_3KEY)
tdes._lib.tdes_get_strace.argtypes = [ctypes.c_void_p]
for n in [int(a) for a in sys.argv[1:]] or (1024, 1 << 17):
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda"); tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    for _ in range(3):
        tdes.ecb_crypt_mode(x, s, 2, out=y)
    torch.cuda.synchronize()
    buf = np.zeros((8, 2, 100), dtype=np.int64)
    tdes._lib.tdes_get_strace(buf.ctypes.data)
    arr, rel = buf[:, 0, :48], buf[:, 1, :48]
    t0 = rel[:, 0].min()
    round_time = np.diff(rel.max(axis=0))
    work = arr[:, 1:] - rel[:, :-1]          # per warp: release(r-1) -> arrival(r)
    wait = rel[:, 1:] - arr[:, 1:]
    print(f"n={n}: cycles per round median {np.median(round_time):.0f} (min {round_time.min()} max {round_time.max()})")
    print("  per-warp work (release->arrival) median by S-box:", [int(np.median(work[g])) for g in range(8)])
    print("  barrier release latency after last arrival, median:", int(np.median(rel.max(axis=0)[1:] - arr.max(axis=0)[1:])))
