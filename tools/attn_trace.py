"""Per-step handoff timeline of CTA 0 in the prefix-prefill kernel (two-tile items).

Needs a trace build:
    make -C paper_2404_12457_b200/csrc BUILD=build_tr OUT=../libragcache_b200_tr.so EXTRA=-DRCB_TRACE
then
    RCB_LIB_PATH=$PWD/paper_2404_12457_b200/libragcache_b200_tr.so TRACE_CASE=long python tools/attn_trace.py

Events (clock64 on the SM of CTA 0; see the TRACE comment in prefix_attn.cu):
softmax WG w, tile c: S-wait start, S seen, P arrive; MMA step s: P0 seen, QK0 issued,
P1 seen, QK1 issued.  Use a case whose items are all pairs with n0 == n1 ("long") so the
WG tile index equals the KV step.
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_12457_b200 import _lib, kernels  # noqa: E402

EV = 16
TILES = 1024


def main():
    lib = _lib.load()
    fn = lib.rcb_debug_attn_trace
    fn.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    case = os.environ.get("TRACE_CASE", "long")
    hq, hkv, bt, hd, L = 32, 8, 64, 128, 2
    reqs = {"long": [(4096, 256)] * 32, "miss": [(0, 1056)] * 16,
            "hit": [(1024, 32)] * 64, "decode": [(4096, 1)] * 64}[case]
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
    tr = buf.reshape(TILES, EV).astype(np.float64)
    mine = np.arange(0, plan.n_work, 148)  # CTA 0's items
    if os.environ.get("TRACE_DUMP"):
        np.save(os.environ["TRACE_DUMP"], buf.reshape(TILES, EV))
        print("items", [(int(plan.tiles_q0[i]), int(plan.tiles_q1[i])) for i in mine])
    steps = int(np.maximum(plan.tiles_q0, plan.tiles_q1)[mine].sum())
    n = min(steps, TILES) - 1
    tr = tr[:n]
    t0 = tr[0, 8] if tr[0, 8] else tr[0, 1]
    per_step = (tr[n - 1, 11] - tr[1, 11]) / (n - 2)
    print(f"case {case}: CTA0 items {len(mine)} steps {steps}; cycles per KV step "
          f"{per_step:.0f} (2 tiles = 4 x 128^3 MMAs: 2048 at the nominal tcgen05 rate)")
    for w in (0, 1):
        b = 4 * w
        print(f"  WG{w}: S wait (start->seen) {np.median(tr[1:, b + 1] - tr[1:, b]):6.0f}   "
              f"softmax (S seen->P arrive) {np.median(tr[1:, b + 2] - tr[1:, b + 1]):6.0f}   "
              f"P arrive->MMA sees P {np.median(tr[1:, 8 + 2 * w] - tr[1:, b + 2]):6.0f}")
    # chain: P0(s) seen -> QK0(s+1) issued -> S0(s+1) seen by WG0
    print(f"  MMA: P0 seen -> QK0(next) issued {np.median(tr[1:n - 1, 9] - 0 * tr[1:n - 1, 8]) - np.median(tr[1:n - 1, 8]):6.0f} (approx)")
    print(f"  QK0(s) issued -> WG0 sees S0(s) {np.median(tr[1:, 1] - tr[1:, 9]):6.0f}   "
          f"QK1(s) issued -> WG1 sees S1(s) {np.median(tr[1:, 5] - tr[1:, 11]):6.0f}")
    print(f"  MMA: P0 seen -> PV0 issued {np.median(tr[1:, 13] - tr[1:, 8]):6.0f}   "
          f"PV0 issued -> K(s+1) seen {np.median(tr[2:, 12] - tr[1:-1, 13]):6.0f}   "
          f"K seen -> QK0 issued {np.median(tr[2:, 9] - tr[2:, 12]):6.0f}   "
          f"P1 seen -> PV1 issued {np.median(tr[1:, 14] - tr[1:, 10]):6.0f}")
    print(f"  WG0 period {np.median(np.diff(tr[1:, 2])):6.0f}   WG1 period {np.median(np.diff(tr[1:, 6])):6.0f}")
    np.set_printoptions(linewidth=220)
    print("steps 4..9 (cycles rel. to step 4 P0 seen):")
    print((tr[4:10] - tr[4, 8]).astype(np.int64))


if __name__ == "__main__":
    main()
