"""Phase timeline of split-kernel launches (experiment aid; needs tools/exp/strace.so
from split_trace_build.py): CTA 0's warps at entry / after the key table / after the
tile load / after the 48 rounds / after the store / exit (%globaltimer), and the
spread of CTA entry and exit times over the grid, for launches queued behind a
device-side sleep (the event pair then times the GPU's own launch processing).

  TDES_LIB_PATH=tools/exp/strace.so python tools/exp/split_phases.py [nblocks ...]
"""
import ctypes
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import paper_2007_10752_b200 as tdes  # noqa: E402
import synthetic  # noqa: E402

lib = tdes._lib
lib.tdes_get_sphase.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
s = tdes.key_schedule(*synthetic.KEYS_3KEY)
names = ["keys", "load", "rounds", "store", "exit"]
for n in [int(a) for a in sys.argv[1:]] or (1024, 16384, 131072):
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda"); tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    for _ in range(3):
        tdes.ecb_crypt_mode(x, s, 2, out=y)
    torch.cuda.synchronize()
    rows = []
    for rep in range(5):
        torch.cuda._sleep(400_000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); tdes.ecb_crypt_mode(x, s, 2, out=y); b.record(); b.synchronize()
        ph = np.zeros((8, 6), dtype=np.uint64); cta = np.zeros((1024, 2), dtype=np.uint64)
        lib.tdes_get_sphase(ph.ctypes.data, cta.ctypes.data)
        ntiles = (n + 1023) // 1024
        c = cta[:min(ntiles, 1024)].astype(np.int64)
        t0 = c[:, 0].min()
        p = (ph.astype(np.int64) - t0) / 1e3
        rows.append((a.elapsed_time(b) * 1e3, p, (c[:, 0].max() - t0) / 1e3, (c[:, 1].min() - t0) / 1e3, (c[:, 1].max() - t0) / 1e3))
    ev, p, ent, ex0, ex1 = sorted(rows, key=lambda r: r[0])[len(rows) // 2]
    steps = " ".join(f"{nm} {np.median(p[:, i + 1] - p[:, i]):5.2f}" for i, nm in enumerate(names))
    print(f"n={n:7d} event {ev:6.1f} us | CTA0 entry {np.median(p[:, 0]):5.2f}, {steps} | "
          f"CTA entries spread {ent:5.2f} us, exits {ex0:6.2f}..{ex1:6.2f} us", flush=True)
