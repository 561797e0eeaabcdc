"""Per-tile timeline of the throughput kernel at mid sizes (experiment aid).

TDES_LIB_PATH=tools/exp/trace.so python tools/exp/trace_tiles.py
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
lib.tdes_set_trace.argtypes = [ctypes.c_void_p]
s = tdes.key_schedule(*synthetic.KEYS_3KEY)
for e in (int(a) for a in (sys.argv[1:] or ["19", "20", "21", "22", "23"])):
    n = 1 << e
    ntiles = n // 1024
    x = torch.empty(8 * n, dtype=torch.uint8, device="cuda"); tdes.fill_splitmix64(x)
    y = torch.empty_like(x)
    tr = torch.zeros(4 * ntiles, dtype=torch.int64, device="cuda")
    lib.tdes_set_trace(0)
    for _ in range(3):
        tdes.ecb_crypt_mode(x, s, 1, out=y)
    lib.tdes_set_trace(tr.data_ptr())
    tdes.ecb_crypt_mode(x, s, 1, out=y)
    torch.cuda.synchronize()
    lib.tdes_set_trace(0)
    t = tr.view(-1, 4).cpu().numpy().astype(np.int64)
    t0 = t[:, 0].min()
    st, en = (t[:, 0] - t0) / 1e3, (t[:, 1] - t0) / 1e3
    dur = en - st
    per_sm = {}
    for i in range(ntiles):
        per_sm.setdefault(int(t[i, 2]), []).append(en[i])
    sm_end = np.array([max(v) for v in per_sm.values()])
    print(f"2^{e}: tiles {ntiles} span {en.max():.1f} us; tile dur min/med/max {dur.min():.1f}/{np.median(dur):.1f}/{dur.max():.1f} us; "
          f"SM end min/med/max {sm_end.min():.1f}/{np.median(sm_end):.1f}/{sm_end.max():.1f}; start max {st.max():.1f}; "
          f"tiles/SM {ntiles/len(per_sm):.1f} on {len(per_sm)} SMs")
