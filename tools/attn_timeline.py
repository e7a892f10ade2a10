"""Item-boundary timeline of CTA 0 in the prefix-prefill kernel (trace build).

    make -C paper_2404_12457_b200/csrc BUILD=build_tr OUT=../libragcache_b200_tr.so EXTRA=-DRCB_TRACE
    RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_tr.so \
        TL_CASE=mistral_miss python tools/attn_timeline.py

For every KV step s of CTA 0 (item, step-in-item j): producer (ids loaded, K issued,
V issued), MMA (K seen, QK0/QK1 issued, P0/P1 seen, PV0/PV1 issued) and, per item, the
epilogue (O0 full seen / freed, O1 full seen / freed, stores done), in cycles relative to
the first event.  Summary: median cycles per step inside items vs across item
boundaries, which is the per-item overhead.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_12457_b200 import _lib, kernels  # noqa: E402

EV = 32
TILES = 1024
CASES = {
    "mistral_miss": (32, 8, [(0, 1056)] * 16),
    "mistral_mixed": (32, 8, [(0, 1056)] * 26 + [(512, 544)] * 26 + [(1024, 32)] * 12),
    "mistral_long": (32, 8, [(4096, 256)] * 32),
    "llama2_miss": (32, 32, [(0, 544)] * 16),
}


def main():
    lib = _lib.load()
    fn = lib.rcb_debug_attn_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    case = os.environ.get("TL_CASE", "mistral_miss")
    rope_on = os.environ.get("TL_ROPE", "0") == "1"
    hq, hkv, reqs = CASES[case]
    bt, hd, L = 64, 128, 2
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
    rope = kernels.rope_table(plan.max_pos + 1, hd, 1e6) if rope_on else None
    for _ in range(3):
        kernels.prefix_prefill(q, o, plan, pool.data_ptr(), nb, block_tokens=bt, n_layers=L,
                               n_kv_heads=hkv, head_dim=hd, layer=1, rope=rope, n_q_heads=hq)
    torch.cuda.synchronize()
    buf = np.zeros(TILES * EV, dtype=np.int64)
    assert fn(buf.ctypes.data, buf.nbytes) == 0
    tr = buf.reshape(TILES, EV).astype(np.float64)
    mine = np.arange(0, plan.n_work, 148)
    n0 = plan.tiles_q0[mine]
    n1 = plan.tiles_q1[mine]
    nsteps = np.maximum(n0, n1)
    t0 = tr[0, 16]
    rel = lambda x: int(x - t0) if x else -1  # noqa: E731
    print(f"case {case} rope={rope_on}: CTA0 items {len(mine)} steps {int(nsteps.sum())}")
    print("item  j  | ids   K_iss  V_iss | K_seen QK0    QK1    P0_seen PV0    P1_seen PV1  | "
          "S0seen P0arr  S1seen P1arr (pair items with n0 == n1 only) | "
          "O0full O0free O1full O1free Odone")
    same = bool(np.all(n0 == n1))
    s = 0
    qk0 = []
    for ii, n in enumerate(nsteps):
        for j in range(int(n)):
            if s >= TILES:
                break
            r = tr[s]
            line = (f"{ii:4d} {j:2d} | {rel(r[16]):6d} {rel(r[17]):6d} {rel(r[18]):6d} | "
                    f"{rel(r[12]):6d} {rel(r[9]):6d} {rel(r[11]):6d} {rel(r[8]):7d} {rel(r[13]):6d} "
                    f"{rel(r[10]):7d} {rel(r[14]):6d}")
            if same:
                line += f" | {rel(r[1]):6d} {rel(r[2]):6d} {rel(r[5]):6d} {rel(r[6]):6d}"
            if j == n - 1 and ii < TILES:
                e = tr[ii]
                line += f" | {rel(e[19]):6d} {rel(e[20]):6d} {rel(e[21]):6d} {rel(e[22]):6d} {rel(e[23]):6d}"
            print(line)
            qk0.append((ii, j, r[9] if r[9] else r[11]))
            s += 1
    # cycles between consecutive QK issues: within an item vs at an item's first step
    inside, boundary = [], []
    for (i1, j1, t1), (i2, j2, t2) in zip(qk0, qk0[1:]):
        (boundary if j2 == 0 else inside).append(t2 - t1)
    if same:
        k = min(len(qk0), TILES) - 2
        print(f"QK0 issued -> S0 seen median {np.median(tr[1:k, 1] - tr[1:k, 9]):.0f}, "
              f"S0 seen -> P0 arrive (softmax, both chunks) {np.median(tr[1:k, 2] - tr[1:k, 1]):.0f}, "
              f"S1 seen -> P1 arrive {np.median(tr[1:k, 6] - tr[1:k, 5]):.0f}")
    # softmax breakdown (WG 0 and 1): S seen -> chunk 0 in registers -> exp done -> P0 arrive
    # -> chunk 1 in registers -> exp done -> P arrive (tile done)
    k = min(len(qk0), TILES) - 2
    for w in (0, 1):
        t = tr[1:k]
        ok = (t[:, 4 * w + 1] > 0) & (t[:, 24 + 4 * w] > 0) & (t[:, 4 * w + 2] > 0)
        t = t[ok]
        if len(t):
            d = lambda a, b: np.median(t[:, b] - t[:, a])  # noqa: E731
            c1 = t[:, 26 + 4 * w] > 0
            print(f"WG{w} softmax (median cycles, n={len(t)}): S seen -> chunk0 in regs "
                  f"{d(4 * w + 1, 24 + 4 * w):.0f}, -> exp0 done {d(24 + 4 * w, 25 + 4 * w):.0f}, "
                  f"chunk1 ld {np.median(t[c1, 26 + 4 * w] - t[c1, 25 + 4 * w]):.0f} "
                  f"(incl. pack/st/arrive of chunk 0), -> exp1 done "
                  f"{np.median(t[c1, 27 + 4 * w] - t[c1, 26 + 4 * w]):.0f}, -> P arrive "
                  f"{np.median(t[c1, 4 * w + 2] - t[c1, 27 + 4 * w]):.0f}; total {d(4 * w + 1, 4 * w + 2):.0f}")
    print(f"QK-to-QK cycles: inside items median {np.median(inside):.0f} (n={len(inside)}), "
          f"into an item's first step median {np.median(boundary):.0f} (n={len(boundary)})")


if __name__ == "__main__":
    main()
