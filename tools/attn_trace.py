"""Per-tile handoff timeline of CTA 0 in the prefix-prefill kernel.

Needs a trace build:  make -C paper_2404_12457_b200/csrc BUILD=build_tr \
    OUT=../libragcache_b200_tr.so EXTRA=-DRCB_TRACE
then  RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_tr.so python tools/attn_trace.py
Events (clock64 on SM of CTA 0): softmax 0 wait-S, 1 S-full, 2 S loaded, 3 max done,
4 max exchanged, 5 exp done, 6 P-free seen, 7 P-full arrive; MMA 8 QK wait, 9 K-full,
10 S-free, 11 PV wait, 12 P-full seen, 13 V-full.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_12457_b200 import _lib, kernels  # noqa: E402

EV = 16
TILES = 512


def main():
    lib = _lib.load()
    fn = lib.rcb_debug_attn_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    case = os.environ.get("TRACE_CASE", "miss")
    hq, hkv, bt, hd, L = 32, 8, 64, 128, 2
    reqs = {"miss": [(0, 1056)] * 16, "hit": [(1024, 32)] * 64,
            "long": [(0, 4096)] * 4}[case]
    total_slots = sum(-(-(a + b) // bt) for a, b in reqs)
    nb = total_slots + 8
    pool = (torch.randn((nb, L, 2, hkv, bt, hd), device="cuda") * 0.5).to(torch.bfloat16)
    perm = np.random.default_rng(0).permutation(nb)
    requests, pos = [], 0
    for a, b in reqs:
        n = -(-(a + b) // bt)
        blocks = [int(x) for x in perm[pos:pos + n]]
        pos += n
        requests.append((b, a, blocks, [bt] * (n - 1) + [a + b - (n - 1) * bt]))
    T = sum(b for _, b in reqs)
    q = torch.randn((T, hq, hd), device="cuda").to(torch.bfloat16)
    o = torch.empty_like(q)
    plan = kernels.AttnPlan(requests, block_tokens=bt, n_q_heads=hq, n_kv_heads=hkv)
    for _ in range(3):
        kernels.prefix_prefill(q, o, plan, pool.data_ptr(), nb, block_tokens=bt, n_layers=L,
                               n_kv_heads=hkv, head_dim=hd, layer=1)
    torch.cuda.synchronize()
    buf = np.zeros(TILES * EV, dtype=np.int64)
    assert fn(buf.ctypes.data, buf.nbytes) == 0
    tr = buf.reshape(TILES, EV)
    items = plan.work_host[0::148]  # CTA 0's items
    n_tiles = int(items[:, 7].sum())
    n = min(n_tiles, TILES)
    tr = tr[:n:2].astype(np.float64)  # softmax WG 0 owns the even tiles
    n = tr.shape[0]
    t0 = tr[0, 0]
    print(f"case {case}: CTA0 items {len(items)} tiles {n_tiles}; total "
          f"{(tr[n - 1, 7] - t0):.0f} cyc, per tile {(tr[n - 1, 7] - t0) / n:.0f}")
    names = {1: "S-full wait", 2: "tmem ld ch0", 3: "max ch0", 4: "-", 5: "rest of tile",
             6: "-", 7: "fence"}
    tr[:, 4] = tr[:, 3]
    tr[:, 6] = tr[:, 5]
    d = np.diff(tr[:, :8], axis=1)
    for k in range(1, 8):
        print(f"  softmax {names[k]:12s} median {np.median(d[:, k - 1]):7.0f}  mean {np.mean(d[:, k - 1]):7.0f}")
    print(f"  softmax period (7->7)    median {np.median(np.diff(tr[:, 7])):7.0f}")
    print(f"  MMA K-full wait          median {np.median(tr[:, 9] - tr[:, 8]):7.0f}")
    print(f"  MMA S-free wait          median {np.median(tr[:, 10] - tr[:, 9]):7.0f}")
    print(f"  MMA P-full wait          median {np.median(tr[:, 12] - tr[:, 11]):7.0f}")
    print(f"  MMA V-full wait          median {np.median(tr[:, 13] - tr[:, 12]):7.0f}")
    print(f"  P-full arrive -> MMA sees median {np.median(tr[:, 12] - tr[:, 7]):7.0f}")
    print(f"  PV issue(g) -> S-full(g+2) seen by softmax median "
          f"{np.median(tr[2:, 1] - tr[:-2, 13]):7.0f}")
    print(f"  QK issue(g) -> S-full(g) seen median {np.median(tr[:, 1] - tr[:, 10]):7.0f}")
    np.set_printoptions(linewidth=200)
    print("first 12 tiles (cycles rel. to tile 0 start):")
    print((tr[:12, :14] - t0).astype(np.int64))


if __name__ == "__main__":
    main()
