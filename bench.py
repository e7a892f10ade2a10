"""Hot-path benchmark: RAG req/s through retrieval + KV tiering + prefix prefill.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload mistral7b-100k] [--batch R]

One step = one batch of R requests per GPU (BASELINE.json configs[1] by
default: Mistral-7B attention shape, 100K-doc 768-d corpus, top-2 x 512-token
docs, Zipf popularity) through the GPU hot path:

  retrieval   staged exact top-k for the R query embeddings (corpus sharded
              over the ranks; NCCL all-gather of queries and of per-shard
              top-k lists, on-device merge)
  tiering     the step's knowledge-tree transitions (reference decisions,
              planned ahead on a shadow pool) replayed on the device pool:
              swap-out D2H / swap-in H2D of KV blocks, suffix block reservation
  prefill     32 layers x (RoPE + paged KV write, prefix-aware attention)

`value` times planned steps (device work only, inputs resident).  `e2e`
times live steps through the public HotPath API: host query buffers copied
H2D, reference tree decisions on the host, block tables uploaded, staged ids
and last-token outputs copied D2H.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import threading
import subprocess
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "p50 TTFT (ms) and RAG req/s vs cache hit rate at 1/2/4/8 B200; KV swap GB/s"


def WORKLOAD_NAMES():
    from paper_2404_12457_b200.workloads import WORKLOADS

    return set(WORKLOADS)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="mistral7b-100k")
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--cache-warm-steps", type=int, default=40)
    ap.add_argument("--swap-mode", type=int, default=0)
    ap.add_argument("--layers-per-group", type=int, default=1,
                    help="a step's swaps are issued per group of this many layers and each "
                         "layer's K/V write + attention waits only for its group (0: the whole "
                         "batch before the prefill)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ttft", action="store_true")
    ap.add_argument("--no-hit-sweep", action="store_true",
                    help="skip the hot-path req/s vs hit rate sweep (part of the ttft block)")
    ap.add_argument("--no-model-step", action="store_true",
                    help="skip timing the bench step's batch through the whole random-init model")
    ap.add_argument("--no-timed", action="store_true",
                    help="skip the hardware-in-the-loop TTFT / req/s curves")
    # multi-rank smoke on a single GPU (all ranks on cuda:0, gloo, small tier)
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"])
    ap.add_argument("--single-device", action="store_true")
    ap.add_argument("--gpu-tier-tokens", type=int, default=0)
    ap.add_argument("--ref-sample", type=int, default=1,
                    help="requests per step timed through the reference CPU path")
    return ap.parse_args()


# ---------------------------------------------------------------------- distributed
from paper_2404_12457_b200.dist import Dist, route, shard_bounds  # noqa: E402


# ---------------------------------------------------------------------- clocks
class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: an NVML thread at
    ~5 ms (the timed region can be a fraction of a second), nvidia-smi as fallback."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40),
               ("sw_thermal_slowdown", 0x20), ("sw_power_cap", 0x4))

    def __init__(self, index: int):
        self.index = index
        self.samples: list[tuple[float, int]] = []
        self.smax = None
        self.thread = None
        self.stop_flag = threading.Event()
        self.error = None

    def start(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.smax = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            get_reasons = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                pynvml.nvmlDeviceGetCurrentClocksThrottleReasons

            def sample():
                self.samples.append((float(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)),
                                     int(get_reasons(h))))

            sample()  # NVML is live before the timed region starts

            def loop():
                while not self.stop_flag.wait(0.005):
                    sample()

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
        except Exception as exc:  # no NVML: the caller still gets a line, marked
            self.error = f"nvml unavailable: {exc}"[:80]

    def stop(self) -> dict:
        if self.thread is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.error or "no samples"]}
        self.stop_flag.set()
        self.thread.join()
        loaded = self.samples[1:] or self.samples  # drop the pre-region sample
        reasons = sorted({n for _, r in loaded for n, bit in self.REASONS if r & bit})
        return {"sm_mhz": statistics.median(c for c, _ in loaded), "sm_max_mhz": self.smax,
                "reasons": reasons, "samples": len(loaded), "source": "nvml, 5 ms"}


NCU_TAG = "r2o"  # profiles/<tag>_ncu_summary.json: captures of the current kernels
E2E_WARM = 2  # untimed live steps before the e2e timing


def ncu_traffic(capture: str):
    """dram__bytes_read.sum + dram__bytes_write.sum of one captured launch, or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                        f"{NCU_TAG}_ncu_summary.json")
    try:
        k = json.load(open(path))["kernels"][capture]
        return float(k["dram_traffic_bytes"]), f"ncu --set full, {os.path.basename(path)}:{capture}"
    except (OSError, KeyError, ValueError):
        return None, None


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        p = json.load(open(path))
        return p["hbm_gbs"], p.get("bf16_tflops_sustained", p["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1400.0, "fallback (B200_PROFILING.md)"


def guarded(fn, *a, **kw):
    """A side measurement (model step, TTFT curves) that fails records the error in its
    block instead of losing the bench line."""
    try:
        return fn(*a, **kw)
    except Exception as exc:  # noqa: BLE001
        torch.cuda.empty_cache()
        return {"error": f"{type(exc).__name__}: {exc}"[:300]}


def burst_frac(achieved_tf: float, clk: dict):
    try:
        p = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        scale = float(clk["sm_mhz"]) / float(p.get("sm_max_mhz") or clk["sm_max_mhz"])
        return round(achieved_tf / (float(p["bf16_tflops"]) * scale), 4)
    except Exception:
        return None


# ---------------------------------------------------------------------- setup
def build_workload(args, dist: Dist):
    from paper_2404_12457_b200 import synth
    from paper_2404_12457_b200.workloads import WORKLOADS, make_stream

    w = WORKLOADS[args.workload]
    R = args.batch or w.batch
    # cache warm-up + warmup + timed (planned) steps, then K fresh steps for e2e
    n_steps = args.cache_warm_steps + args.warmup + 2 * args.steps + E2E_WARM
    n_req = n_steps * R * dist.world
    trace, sizes = make_stream(w, n_req, rate=1.0)
    mine = route(trace, dist.rank, dist.world)  # DP routing: id mod G
    steps = [mine[i * R:(i + 1) * R] for i in range(n_steps)]
    # corpus shard of this rank (global ids [lo, hi)); queries from the targets' rows
    lo, hi = shard_bounds(w.num_docs, dist.rank, dist.world)
    return w, R, steps, sizes, (lo, hi)


def make_queries(w, batch_reqs, rows: int | None = None):
    """Query embeddings of a step's requests, zero-padded to `rows` (fixed retrieval batch)."""
    from paper_2404_12457_b200 import synth

    docs = [r.doc_sequence for r in batch_reqs]
    q = synth.build_queries(lambda ids: synth.corpus_rows(ids, synth.EMB_DIM, w.seed), docs,
                            seed=batch_reqs[0].id if batch_reqs else 0)
    if rows is not None and q.shape[0] < rows:
        q = np.concatenate([q, np.zeros((rows - q.shape[0], synth.EMB_DIM))])
    return torch.from_numpy(q.astype(np.float32)).to(torch.bfloat16)


def fence_step(dpool, compute, swapped: bool, layers_per_group: int):
    """Issue the step's pending swaps and order the prefill after them.  With swaps and
    layers_per_group > 0 they go out per layer group (swap-outs off the critical path:
    layer l's K/V write waits only for the swap-outs' layer-l slices of the blocks it
    reuses, simulator.py:505-507); returns the per-layer fence for HotPath.prefill."""
    if swapped and layers_per_group > 0:
        dpool.flush_layered(layers_per_group)
        return lambda layer: dpool.fence_layer(layer, compute)
    dpool.fence_into(compute)
    return None


def run_ours(args, dist: Dist, emit: bool = True):
    from paper_2404_12457_b200 import _lib, synth
    from paper_2404_12457_b200.hotpath import HotPath, StepPlan, apply_events, EventLog, has_swaps
    from paper_2404_12457_b200.pool import accounting_pool
    from paper_2404_12457_b200.retrieval import ShardedRetriever
    from paper_2404_12457_b200.workloads import pool_blocks

    torch.cuda.set_device(0 if args.single_device else dist.local)
    if dist.pg is None:  # a hit-rate sweep run reuses the process group
        dist.init(args.backend)
    dist.device = "cuda"
    w, R, steps, sizes, (lo, hi) = build_workload(args, dist)
    raw_steps = list(steps)  # the planning loop below keeps only each step's admitted prefix
    if args.gpu_tier_tokens:
        import dataclasses as _dc

        w = _dc.replace(w, gpu_capacity_tokens=args.gpu_tier_tokens)
    shape = w.model
    ng = pool_blocks(w.gpu_capacity_tokens, w.block_tokens, sizes.values(), R * (w.k + 1))
    nh = pool_blocks(w.host_capacity_tokens, w.block_tokens, sizes.values(), 0)
    profile, profile_src = tree_profile(w)
    copy_stream = torch.cuda.Stream()
    compute = torch.cuda.current_stream()

    # shadow planner (accounting-only pool) and the device replica
    shadow_pool = EventLog(accounting_pool(ng, nh, w.block_tokens))
    planner = HotPath(shape, gpu_capacity_tokens=w.gpu_capacity_tokens,
                      host_capacity_tokens=w.host_capacity_tokens, block_tokens=w.block_tokens,
                      num_gpu_blocks=ng, num_host_blocks=nh, sizes=sizes, profile=profile,
                      pool=shadow_pool)
    device = HotPath(shape, gpu_capacity_tokens=w.gpu_capacity_tokens,
                     host_capacity_tokens=w.host_capacity_tokens, block_tokens=w.block_tokens,
                     num_gpu_blocks=ng, num_host_blocks=nh, sizes=sizes, profile=profile,
                     swap_mode=args.swap_mode, copy_stream=copy_stream)
    dpool = device.pool

    n_warm = args.cache_warm_steps
    n_planned = n_warm + args.warmup + args.steps
    plans = []
    t_plan = time.perf_counter()
    hits = total = 0
    carry = []
    for i, batch in enumerate(steps[:n_planned]):
        # requests that did not fit the previous step (pinned/reserved capacity) go first
        batch = carry + list(batch)
        cand, rest = batch[:R], batch[R:]
        adm = planner.admit_batch([(r.id, r.doc_sequence, r.prompt_tokens) for r in cand])
        if not adm:
            raise RuntimeError("a single request exceeds the GPU tier's evictable capacity")
        carry = cand[len(adm):] + rest
        steps[i] = cand[:len(adm)]
        ev = shadow_pool.take()
        for a in adm:
            planner.commit(a)
        cev = shadow_pool.take()
        plan = StepPlan(adm, ev, cev)
        if i < n_warm:
            apply_events(dpool, ev)
            apply_events(dpool, cev)
        else:
            plans.append(plan)
            hits += sum(len(a.matched) for a in adm)
            total += sum(len(a.docs) for a in adm)
    plan_s = time.perf_counter() - t_plan
    dpool.sync()
    for p in plans:
        device.prepare_device(p)
    hit_rate = hits / max(1, total)

    # corpus shard + per-step queries (resident)
    corpus = synth.corpus_device(hi - lo, seed=w.seed, row_offset=lo)
    retr = ShardedRetriever(corpus, lo, w.k, w.n_stages, dist, batch=R)
    qs = [make_queries(w, steps[n_warm + i], R).cuda() for i in range(len(plans))]
    # worst case suffix rows of a step: every doc missed
    max_t = R * (w.k * max(sizes.values()) + w.prompt_tokens)
    g = torch.Generator(device="cuda")
    g.manual_seed(1234 + dist.rank)
    qkv = (torch.randn((max_t, shape.qkv_width), generator=g, device="cuda") * 0.5).to(torch.bfloat16)
    q_rot = None  # Q's RoPE is fused into the attention kernel
    out = torch.empty((max_t, shape.n_q_heads, shape.head_dim), dtype=torch.bfloat16, device="cuda")

    def device_step(i, attn_events=None, scan_events=None):
        p = plans[i]
        if scan_events is not None:
            scan_events.append((torch.cuda.Event(enable_timing=True),
                                torch.cuda.Event(enable_timing=True)))
            scan_events[-1][0].record()
        ids = retr(qs[i])
        if scan_events is not None:
            scan_events[-1][1].record()
        apply_events(dpool, p.events)
        fence = fence_step(dpool, compute, has_swaps(p.events), args.layers_per_group)
        device.prefill(p, qkv, q_rot, out, events=attn_events, layer_fence=fence)
        dpool.wait_for(compute)
        apply_events(dpool, p.commit_events)
        return ids

    # ---- warmup (untimed), then the timed K steps
    W, K = args.warmup, args.steps
    for i in range(W):
        device_step(i)
    torch.cuda.synchronize()
    # correctness at full size: every timed step's final stage equals the ground truth
    retrieval_exact = True
    for i in range(W, W + K):
        want = np.array([r.doc_sequence for r in steps[n_warm + i]], dtype=np.int64)
        final = retr(qs[i])[: len(want), -1].cpu().numpy()
        retrieval_exact &= bool(np.array_equal(final, want))

    attn_ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
                for _ in range(shape.n_layers)] for _ in range(K)]
    scan_ev = []
    st0 = dpool.stats()
    launches0 = retr.launches
    clocks = ClockSampler(dist.local)
    dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    c0 = torch.cuda.Event(enable_timing=True)
    c1 = torch.cuda.Event(enable_timing=True)
    t0.record()
    c0.record(copy_stream)
    for i in range(K):
        device_step(W + i, attn_events=attn_ev[i], scan_events=scan_ev)
    dpool.flush()
    c1.record(copy_stream)
    compute.wait_stream(copy_stream)
    t1.record()
    torch.cuda.synchronize()
    clk = clocks.stop()
    elapsed_ms = t0.elapsed_time(t1)
    elapsed_ms = dist.max(elapsed_ms)
    st1 = dpool.stats()
    n_layers = shape.n_layers
    served = dist.sum(float(sum(len(plans[W + i].admissions) for i in range(K))))
    value = served / (elapsed_ms / 1e3)

    # attention roofline (dominant kernel): algorithmic FLOPs per launch / mean launch time
    attn_ms = [a.elapsed_time(b) for evs in attn_ev for a, b in evs]
    flops = [plans[W + i].dev["flops"] for i in range(K) for _ in range(n_layers)]
    hbm_peak, tc_peak, peak_kind = peaks()
    attn_mean_ms = sum(attn_ms) / len(attn_ms)
    achieved_tf = (sum(flops) / len(flops)) / (attn_mean_ms / 1e3) / 1e12
    # algorithmic bytes per launch: KV of alpha+beta tokens for one layer +
    # Q read + O write; traffic = DRAM bytes of the same launch from the committed ncu
    # --set full capture of the bench step (profiles/<tag>_ncu_summary.json, attn_bench)
    attn_bytes = sum(
        sum((a.alpha + a.beta) * 2 * shape.n_kv_heads * shape.head_dim * 2
            + 4 * a.beta * shape.n_q_heads * shape.head_dim for a in plans[W + i].admissions)
        for i in range(K)) / K
    traffic, traffic_src = ncu_traffic("attn_bench")
    scan_ms = [a.elapsed_time(b) for a, b in scan_ev]
    # device time of the step's local scan (every pass: scan + PDL-chained merge) without
    # host launch gaps: the first timed step's gathered queries, replayed back to back
    # from a CUDA graph (corpus >> L2)
    q_block = dist.all_gather(qs[W]).reshape(-1, qs[W].shape[1]) if dist.world > 1 else qs[W]
    dev_scan_ms = retr.device_ms(q_block)
    scan_bytes = retr.bytes_per_scan
    n_passes = len(retr.passes)
    shard_exchange = retr.exchange
    scan_gbs = scan_bytes / (dev_scan_ms / 1e3) / 1e9
    d2h = st1["d2h_bytes"] - st0["d2h_bytes"]
    h2d = st1["h2d_bytes"] - st0["h2d_bytes"]
    copy_ms = c0.elapsed_time(c1)
    kernel_launches = (retr.launches - launches0) + K * 2 * n_layers + \
        (st1["kernel_launches"] - st0["kernel_launches"])

    # ---- the same step with the model around the hot path (paper-sense prefill req/s)
    model_step = (guarded(measure_model_step, w, plans[W], dpool, device)
                  if dist.rank == 0 and not args.no_model_step else None)
    dist.barrier()  # the other ranks wait on the host, not in a peer-exchange spin

    # ---- e2e: live steps through the public API (host buffers, host decisions)
    e2e = run_e2e(args, dist, w, R, steps, planner, device, dpool, retr, qkv, q_rot, out,
                  shadow_pool, compute)

    dpool.close()
    swap = measure_swap(shape) if dist.rank == 0 else None
    ttft = None
    if dist.rank == 0 and not args.no_ttft:
        del corpus, retr, qkv, q_rot, out
        torch.cuda.empty_cache()
        ttft = guarded(measure_ttft, w, swap,
                       stage_ms=(sum(scan_ms) / max(1, len(scan_ms))) / w.n_stages,
                       timed_on=not args.no_timed)

    result = None
    if dist.rank == 0:
        cpu = None if args.no_cpu_baseline or dist.world > 1 else \
            cpu_baseline(args, w, R, raw_steps, sizes, profile, profile_src)
        result = {
            "metric": METRIC,
            "value": round(value, 3),
            "unit": "req/s",
            "n_gpus": dist.world,
            "steps": K,
            "warmup": W,
            "ms_per_step": round(elapsed_ms / K, 3),
            "higher_is_better": True,
            "scaling": "weak",
            "vs_baseline": None,
            "dtype": "bf16",
            "data": "synthetic (ragsim generators: Zipf 0.97 docs x 512 tok; unit-norm "
                    "Irwin-Hall 768-d bf16 embeddings, queries built from the ground-truth "
                    "docs; random bf16 activations in place of model projections)",
            "config": bench_config(w, R, dist.world),
            "tree_profile": profile_src,
            "kv_geometry": {"source_shape": shape.name, "n_layers": shape.n_layers,
                            "n_q_heads": shape.n_q_heads, "n_kv_heads": shape.n_kv_heads,
                            "head_dim": shape.head_dim,
                            "kv_bytes_per_token": shape.kv_bytes_per_token},
            "doc_hit_rate": round(hit_rate, 4),
            "retrieval_final_stage_matches_ground_truth": retrieval_exact,
            "roofline": {
                "kernel": "rcb prefix_prefill (tcgen05)",
                "bound": "tensor",
                "achieved": round(achieved_tf, 2),
                "peak": tc_peak,
                "unit": "TFLOP/s",
                "frac": round(achieved_tf / tc_peak, 4),
                "traffic": traffic,
                "traffic_source": traffic_src,
                "algorithmic_bytes_per_launch": attn_bytes,
                "peak_source": f"{peak_kind} bf16 sustained",
                "launch_ms_mean": round(attn_mean_ms, 4),
                "flops_per_launch": sum(flops) / len(flops),
                "share_of_step": round(sum(attn_ms) / elapsed_ms, 4),
                # the measured burst peak scaled to the clock the step ran at (the kernel is
                # clock-bound under the power cap; burst taken at max clock)
                "frac_of_burst_at_step_clock": burst_frac(achieved_tf, clk),
            },
            "retrieval": {"device_ms": round(dev_scan_ms, 4),
                          "achieved_gbs": round(scan_gbs, 1), "peak_gbs": hbm_peak,
                          "frac": round(scan_gbs / hbm_peak, 4),
                          "call_ms_mean": round(sum(scan_ms) / max(1, len(scan_ms)), 4),
                          "passes_per_step": n_passes,
                          "shard_exchange": shard_exchange,
                          "how": "device_ms: the first timed step's queries, 20 local scans "
                                 "(scan + merge kernels per pass) replayed from a CUDA graph, "
                                 "CUDA events; call_ms_mean: in-step event pair around the "
                                 "retrieval call (gathers, scans, merge; includes launch gaps)"},
            "kv_swap": swap,
            "step_swap_bytes": {"d2h": d2h, "h2d": h2d},
            "plan_host_s": round(plan_s, 3),
            "e2e": e2e,
            "model_step": model_step,
            "ttft": ttft,
            "gpu_launches": int(kernel_launches),
            "clocks": clk,
            "cpu_baseline": cpu,
        }
        if emit:
            print(json.dumps(result))
    return result


SWEEP_TIERS = (80_000, 200_000, 500_000, 1_100_000)


def hit_rate_sweep(args, dist: Dist) -> dict:
    """The hot-path step's req/s against the cache hit rate (BASELINE metric: "RAG req/s vs
    cache hit rate"): the repeated-question variant of the workload (ragsim query pool) over
    GPU tiers from barely above the batch's in-flight need to configs[1]'s, same batch and
    step, fewer steps; every point a full run_ours (device-timed steps + e2e)."""
    import copy

    t0 = time.perf_counter()
    pts = []
    for tier in SWEEP_TIERS:
        a = copy.copy(args)
        a.workload, a.gpu_tier_tokens = args.workload + "-qpool", tier
        a.no_ttft = a.no_cpu_baseline = a.no_model_step = True
        a.steps, a.warmup = 5, 3
        torch.cuda.empty_cache()
        try:
            r = run_ours(a, dist, emit=False)
        except Exception as exc:  # noqa: BLE001 - a failed point must not lose the main line
            pts.append({"gpu_tier_tokens": tier, "error": f"{type(exc).__name__}: {exc}"[:300]})
            continue
        pts.append({"gpu_tier_tokens": tier, "doc_hit_rate": r["doc_hit_rate"],
                    "req_per_s": r["value"], "e2e_req_per_s": r["e2e"]["value"],
                    "e2e_doc_hit_rate": r["e2e"]["doc_hit_rate"],
                    "ms_per_step": r["ms_per_step"], "attention_frac": r["roofline"]["frac"]})
    from paper_2404_12457_b200.workloads import WORKLOADS

    return {"workload": args.workload + "-qpool",
            "batch_per_gpu": args.batch or WORKLOADS[args.workload + "-qpool"].batch,
            "points": pts, "seconds": round(time.perf_counter() - t0, 1),
            "how": "each point: bench.py's step (retrieval + KV tiering + K/V write + attention) "
                   "at that GPU tier, 40 cache-warm + 3 warmup + 5 device-timed steps, e2e "
                   "through HotPath; hits rise with the tier because the repeated questions' "
                   "documents stay resident"}


def measure_model_step(w, plan, dpool, device, reps: int = 2) -> dict:
    """The first timed step's admissions (same block tables, same pool) through the whole
    random-init model: QKV / O / MLP library GEMMs and the fused RMSNorm / SiLU kernels around
    the hot path's K/V write + prefix attention, every layer (model.PrefillModel).  This is the
    prefill work a serving step does for those requests; `value` covers only the hot path."""
    from paper_2404_12457_b200.model import DIMS, PrefillModel, init_weights

    dims = DIMS.get(w.shape)
    if dims is None:
        return {"skipped": f"no model dims for {w.shape}"}
    d = plan.dev
    T = int(d["pos"].shape[0])
    free, _ = torch.cuda.mem_get_info()
    s = dims.shape
    hd = dims.d_model
    need = (2 * (dims.vocab * hd * 2 + s.n_layers * (
        hd * (s.qkv_width + s.n_q_heads * s.head_dim)
        + dims.ffn * hd * 3 * max(1, dims.n_experts)))  # bf16 weights
        + T * (hd * 16 + dims.ffn * 4 * max(1, dims.top_k)) + (4 << 30))  # activations + slack
    if free < need:
        return {"skipped": f"needs ~{need / 2**30:.0f} GiB next to the pool, {free / 2**30:.0f} free"}
    wts = init_weights(dims, seed=0)
    model = PrefillModel(dims, wts, block_tokens=w.block_tokens, num_pool_blocks=dpool.num_gpu_blocks,
                         pool_base=dpool.gpu_base)
    g = torch.Generator(device="cuda")
    g.manual_seed(7)
    tokens = torch.randint(0, dims.vocab, (T,), generator=g, device="cuda")
    run = lambda: model.prefill(tokens, d["pos"], d["slots"], d["attn"], d["last"])  # noqa: E731
    run()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        logits = run()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    ms = float(np.median(ts))
    n = len(plan.admissions)
    out = {"req_per_s": round(n / ms * 1e3, 2), "ms_per_step": round(ms, 3), "requests": n,
           "suffix_tokens": T, "logits_finite": bool(torch.isfinite(logits).all()),
           "how": f"the first timed step's {n} admissions (same block tables and pool) through "
                  f"the whole random-init {w.shape} model: cuBLAS QKV/O/MLP GEMMs + rcb "
                  f"RMSNorm/SiLU, K/V write and prefix attention per layer; CUDA events, "
                  f"median of {reps}"}
    del model, wts
    torch.cuda.empty_cache()
    return out


def measure_timed(w, qw, prof, decode_ms, stage_ms, pcie, max_rate: float = 400.0) -> dict:
    """Hardware-in-the-loop curves (every admitted prefill executed on the GPU, TimedEngine):
    TTFT vs hit rate over 4 GPU tiers and req/s at the 5x TTFT SLO on the repeated-question
    variant of this workload, plus configs[2] (LLaMA2-7B top-5, two tiers) with real
    layer-pipelined swaps."""
    import tempfile

    from ragsim.cost_model import save_profile_csv

    from paper_2404_12457_b200.timed_curves import (TimedRunner, timed_slo_throughput,
                                                    timed_ttft_curve)
    from paper_2404_12457_b200.workloads import WORKLOADS

    out = {"engine": "TimedEngine: ragsim decisions/queue/DSP/virtual clock; every admitted "
                     "prefill run on the GPU (random-init model: cuBLAS GEMMs + rcb kernels on "
                     "its block table) and its CUDA-event time advances the clock"}
    t0 = time.perf_counter()
    with tempfile.TemporaryDirectory() as td:
        path = os.path.join(td, "profile.csv")
        save_profile_csv(prof, path)
        if qw is not None:
            floor = qw.k * int(qw.doc_tokens_mean) + qw.prompt_tokens + 64
            tiers = sorted({max(floor, t) for t in (2200, 55_000, 220_000, 440_000)})
            runner = TimedRunner(qw, max(tiers), qw.host_capacity_tokens)
            kw = dict(prof_path=path, dec_ms=decode_ms, stage_ms=stage_ms, pcie_gbs=pcie)
            out["vs_hit_rate"] = {"workload": qw.name, "requests": 400, "rate_req_s": 2.0,
                                  "points": timed_ttft_curve(runner, tiers, n_requests=400, **kw)}
            out["req_per_s_at_5x_slo"] = {
                "workload": qw.name, "how": "ragsim's measure_throughput bisection "
                "(simulator.py:648-681), every probe a timed run",
                "points": [timed_slo_throughput(runner, cap, n_requests=300, max_rate=max_rate, **kw)
                           for cap in (tiers[0], tiers[-1])]}
            runner.close()
    c2 = WORKLOADS["llama2-7b-top5-qpool"]
    c2_prof = os.path.join(ROOT, "profiles", f"{c2.shape}_b200_profile.csv")
    if os.path.exists(c2_prof):
        info = json.load(open(c2_prof.replace(".csv", ".json")))
        runner = TimedRunner(c2, c2.gpu_capacity_tokens, c2.host_capacity_tokens,
                             swap_in="layered")
        pts = timed_ttft_curve(runner, [c2.gpu_capacity_tokens], prof_path=c2_prof,
                               dec_ms=float(info["decode_ms_per_token"]["2592"]),
                               stage_ms=stage_ms, pcie_gbs=pcie, n_requests=240, rate=1.0)
        runner.close()
        out["configs2_two_tier"] = {"workload": c2.name, "gpu_tier_tokens": c2.gpu_capacity_tokens,
                                    "host_tier_tokens": c2.host_capacity_tokens,
                                    "swap_in": "layer-pipelined (executed)", **pts[0]}
    out["seconds"] = round(time.perf_counter() - t0, 1)
    return out


def measure_ttft(w, swap, stage_ms: float, timed_on: bool = True) -> dict:
    """p50 TTFT on B200 costs: measure T(alpha, beta) of the real prefill (our kernels +
    cuBLAS GEMMs, CUDA-graph replay), then run the reference engine (ragsim, decisions
    unchanged) on this workload and on its repeated-question variant across GPU tiers."""
    from paper_2404_12457_b200.profile import decode_ms_per_token, measure_profile
    from paper_2404_12457_b200.ttft import slo_throughput, ttft_curve
    from paper_2404_12457_b200.workloads import WORKLOADS

    t0 = time.perf_counter()
    prof, info = measure_profile(w.shape, block_tokens=w.block_tokens, reps=3)
    t_prof = time.perf_counter() - t0
    pcie = swap["h2d_gbs"] if swap else 55.0
    # decode step cost at the workload's typical context (k docs + prompt)
    ctx = w.k * int(w.doc_tokens_mean) + w.prompt_tokens
    decode_ms = decode_ms_per_token(prof, ctx)
    own = ttft_curve(w, prof, gpu_tiers=[w.gpu_capacity_tokens], host_tier=w.host_capacity_tokens,
                     n_requests=2000, pcie_gbs=pcie, stage_interval_ms=stage_ms,
                     decode_ms_per_token=decode_ms)[0]
    qw = WORKLOADS.get(w.name + "-qpool")
    curve, slo, slo_s = [], [], 0.0
    if qw is not None:
        floor = qw.k * int(qw.doc_tokens_mean) + qw.prompt_tokens + 64
        tiers = sorted({max(floor, int(x * qw.gpu_capacity_tokens)) for x in (0.002, 0.05, 0.2, 1.0)})
        curve = ttft_curve(qw, prof, gpu_tiers=tiers, host_tier=qw.host_capacity_tokens,
                           n_requests=2000, pcie_gbs=pcie, stage_interval_ms=stage_ms,
                           decode_ms_per_token=decode_ms)
        t1 = time.perf_counter()
        slo = slo_throughput(qw, prof, gpu_tiers=[tiers[0], tiers[-1]],
                             host_tier=qw.host_capacity_tokens, pcie_gbs=pcie,
                             decode_ms_per_token=decode_ms)
        slo_s = time.perf_counter() - t1
    # the timed bisection's upper bracket: twice the profile-driven rate (its 7 halvings then
    # resolve ~0.5 req/s instead of ~3 from ragsim's default 400 req/s bracket)
    hi = 2.0 * max((p["req_per_s_at_slo"] for p in slo), default=200.0)
    timed = measure_timed(w, qw, prof, decode_ms, stage_ms, pcie, max_rate=hi) if timed_on else None
    idx = {(a, b): prof.times[i][j] for i, a in enumerate(prof.alpha_grid)
           for j, b in enumerate(prof.beta_grid)}
    return {"timed": timed, "p50_ttft_ms": own["p50_ttft_ms"], "mean_ttft_ms": own["mean_ttft_ms"],
            "doc_hit_rate": own["doc_hit_rate"], "engine": "ragsim SimulationEngine (TieredEngine) "
            "on the B200-measured prefill profile and decode step, rate 2 req/s, 2000 requests",
            "retrieval_stage_ms": round(stage_ms, 4),
            "decode_ms_per_token": {"value": round(decode_ms, 3), "context_tokens": ctx,
                                    "replaces": "ragsim RunConfig.decode_ms_per_token = 20.0"},
            "prefill_ms": {"cached1024_new32": round(idx[(1024, 32)], 3),
                           "cached0_new1024": round(idx[(0, 1024)], 3),
                           "cached0_new4096": round(idx[(0, 4096)], 3)},
            "profile": info, "profile_seconds": round(t_prof, 1),
            "req_per_s_at_5x_slo": {"workload": qw.name if qw else None,
                                    "how": "ragsim measure_throughput (simulator.py:648-681) on "
                                           "the B200 profile + decode step",
                                    "points": slo if qw is not None else [],
                                    "seconds": round(slo_s, 1) if qw is not None else None},
            "vs_hit_rate": {"workload": qw.name if qw else None,
                            "points": [{k: r[k] for k in ("gpu_tier_tokens", "doc_hit_rate",
                                                          "p50_ttft_ms", "mean_ttft_ms")}
                                       for r in curve]}}


def measure_swap(shape, n_nodes: int = 64, node_tokens: int = 512) -> dict:
    """KV swap GB/s through the pool (the bench's swap path) against the pinned
    cudaMemcpyAsync peak measured in the same run, plus the HBM gather kernel."""
    from paper_2404_12457_b200 import kernels
    from paper_2404_12457_b200.pool import BlockPool

    hbm_peak, _, _ = peaks()
    n = 1 << 30
    host = torch.empty(n, dtype=torch.uint8).pin_memory()
    dev = torch.empty(n, dtype=torch.uint8, device="cuda")

    def t_copy(fn, reps=5):
        ts = []
        fn()
        for _ in range(reps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            fn()
            b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    pk_h2d = n / t_copy(lambda: dev.copy_(host, non_blocking=True)) / 1e6
    pk_d2h = n / t_copy(lambda: host.copy_(dev, non_blocking=True)) / 1e6
    del host, dev
    bt = 64
    pool = BlockPool(n_nodes * node_tokens // bt + 8, n_nodes * node_tokens // bt + 8,
                     block_tokens=bt, n_layers=shape.n_layers, n_kv_heads=shape.n_kv_heads,
                     head_dim=shape.head_dim)
    keys = list(range(n_nodes))
    for k in keys:
        pool.node_alloc_gpu(k, node_tokens)
    pool.sync()
    t_out, t_in = [], []
    for _ in range(4):
        t0 = time.perf_counter()
        pool.node_swap_out(keys)
        pool.sync()
        t1 = time.perf_counter()
        pool.node_swap_in(keys)
        pool.sync()
        t2 = time.perf_counter()
        for k in keys:
            pool.node_free_host(k)
        t_out.append(t1 - t0)
        t_in.append(t2 - t1)
    nbytes = n_nodes * (node_tokens // bt) * pool.block_bytes
    d2h = nbytes / statistics.median(t_out[1:]) / 1e9
    h2d = nbytes / statistics.median(t_in[1:]) / 1e9
    # HBM gather kernel (the staged path's device half): r+w bytes
    nb = n_nodes * node_tokens // bt
    pairs = torch.tensor([[i, (i * 7919) % nb] for i in range(nb)], dtype=torch.int32, device="cuda")
    scratch = torch.empty(nb * pool.block_bytes, dtype=torch.uint8, device="cuda")
    ms = t_copy(lambda: kernels.block_copy(pool.gpu_base, scratch.data_ptr(), pool.block_bytes, pairs))
    gather = 2 * nb * pool.block_bytes / ms / 1e6
    pool.close()
    return {"path": "staged (gather kernel + cudaMemcpyAsync)", "block_bytes": pool.block_bytes,
            "batch_bytes": nbytes, "d2h_gbs": round(d2h, 2), "h2d_gbs": round(h2d, 2),
            "pcie_peak_d2h_gbs": round(pk_d2h, 2), "pcie_peak_h2d_gbs": round(pk_h2d, 2),
            "frac_d2h": round(d2h / pk_d2h, 4), "frac_h2d": round(h2d / pk_h2d, 4),
            "gather_hbm_gbs": round(gather, 1), "gather_frac_hbm": round(gather / hbm_peak, 4),
            "peak_source": "pinned cudaMemcpyAsync measured in this run; HBM measured peak"}


def run_e2e(args, dist, w, R, steps, planner, device, dpool, retr, qkv, q_rot, out, shadow_pool,
            compute):
    """Live steps: the planner's tree now drives the DEVICE pool directly."""
    from paper_2404_12457_b200.hotpath import StepPlan

    # the shadow tree already mirrors the device pool: hand it the real pool
    planner.pool = dpool
    planner.tree.pool = dpool
    K = args.steps
    n_done = args.cache_warm_steps + args.warmup + args.steps
    # fresh requests (never planned): E2E_WARM untimed live steps first (first-touch costs of
    # the live path: pinned staging, allocator growth), then the K timed ones
    extra = steps[n_done:n_done + E2E_WARM + K]
    host_q = [make_queries(w, b, R).pin_memory() for b in extra]
    q_dev = [torch.empty((R, host_q[0].shape[1]), dtype=torch.bfloat16, device="cuda")
             for _ in range(2)]
    ids_host = [torch.empty((R, w.n_stages, w.k), dtype=torch.int64).pin_memory()
                for _ in range(2)]
    ids_ready = [torch.cuda.Event() for _ in range(2)]
    out_host = torch.empty((R, w.model.n_q_heads, w.model.head_dim),
                           dtype=torch.bfloat16).pin_memory()
    h2d = d2h = 0
    hits = docs_total = 0
    served = 0
    ok = True

    rstream = torch.cuda.Stream()  # retrieval runs beside the prefill stream

    def launch_retrieval(i):
        b = i & 1
        with torch.cuda.stream(rstream):
            q_dev[b].copy_(host_q[i], non_blocking=True)
            ids = retr(q_dev[b])
            ids_host[b].copy_(ids, non_blocking=True)
            ids_ready[b].record(rstream)

    # software pipeline: step i+1's retrieval runs on its own stream while step i's
    # prefill runs, so the host's admissions/commits overlap device work
    launch_retrieval(0)
    carry = []  # (request, retrieved docs) deferred by a full GPU tier: served first next step
    hs = dict.fromkeys(("wait_ids", "admit", "prepare", "launch", "commit"), 0.0)
    pc = time.perf_counter
    for i, batch in enumerate(extra):
        if i == E2E_WARM:
            dpool.sync()
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            h2d = d2h = hits = docs_total = served = 0
            hs = dict.fromkeys(hs, 0.0)
        ta = pc()
        ids_ready[i & 1].synchronize()
        hs["wait_ids"] += pc() - ta
        if i + 1 < len(extra):
            launch_retrieval(i + 1)
        docs = [tuple(int(x) for x in row) for row in ids_host[i & 1][: len(batch), -1].numpy()]
        ok &= docs == [r.doc_sequence for r in batch]
        todo = carry + list(zip(batch, docs))
        cand = todo[:R]
        sw0 = dpool.stats()
        ta = pc()
        adm = planner.admit_batch([(r.id, d, r.prompt_tokens) for r, d in cand])
        tb = pc()
        hs["admit"] += tb - ta
        sw1 = dpool.stats()
        swapped = (sw1["swap_out_calls"], sw1["swap_in_calls"]) != (sw0["swap_out_calls"],
                                                                    sw0["swap_in_calls"])
        carry = todo[len(adm):]
        served += len(adm)
        plan = StepPlan(adm, [], [])
        ta = pc()
        device.prepare_device(plan)
        tb = pc()
        hs["prepare"] += tb - ta
        fence = fence_step(dpool, compute, swapped, args.layers_per_group)
        device.prefill(plan, qkv, q_rot, out, layer_fence=fence)
        dpool.wait_for(compute)
        last = plan.dev["last"]
        out_host[: len(adm)].copy_(out[last], non_blocking=True)
        ta = pc()
        hs["launch"] += ta - tb
        for a in adm:
            planner.commit(a)
        hs["commit"] += pc() - ta
        hits += sum(len(a.matched) for a in adm)
        docs_total += sum(len(a.docs) for a in adm)
        h2d += host_q[i].numel() * 2 + plan.dev["attn"]._buf.numel() * 4 + \
            (plan.dev["pos"].numel() * 2 + plan.dev["last"].numel()) * 4
        d2h += ids_host[0].numel() * 8 + len(adm) * out_host[0].numel() * 2
    dpool.sync()  # the step's swap copies are part of the work
    torch.cuda.synchronize()
    el = time.perf_counter() - t0
    el = dist.max(el)
    served = dist.sum(float(served))
    return {"value": round(served / el, 3), "unit": "req/s", "deferred_at_end": len(carry),
            "doc_hit_rate": round(hits / max(1, docs_total), 4),
            "h2d_bytes_per_step": int(h2d // K), "d2h_bytes_per_step": int(d2h // K),
            "ms_per_step": round(el * 1e3 / K, 3), "retrieval_matches_ground_truth": bool(ok),
            "host_ms_per_step": {k: round(v * 1e3 / K, 3) for k, v in hs.items()},
            "includes": "host ragsim decisions + pool events + planning + H2D/D2H + kernels; "
                        "retrieval on a side stream, host decisions overlap the previous "
                        "step's prefill"}


# ---------------------------------------------------------------------- CPU baselines
def tree_profile(w):
    """PGDSF's cost profile for the bench tree (tree.py:240): the B200-measured T(alpha, beta)
    grid of this model shape (profiles/<shape>_b200_profile.csv, written by profile.py via
    tools/ttft_curve.py), else ragsim's synthetic profile.  Both arms use the same one."""
    from ragsim.cost_model import load_profile_csv, synthetic_profile

    path = os.path.join(ROOT, "profiles", f"{w.shape}_b200_profile.csv")
    if os.path.exists(path):
        return load_profile_csv(path), os.path.relpath(path, ROOT)
    return synthetic_profile(), "ragsim synthetic_profile (no B200 grid committed for this shape)"


def bench_config(w, R: int, world: int) -> dict:
    """The `config` object of both arms (identical by construction)."""
    shard_rows = -(-w.num_docs // world)
    return {
        "workload": w.name,
        "batch_per_gpu": R,
        "corpus_docs": w.num_docs,
        "doc_tokens": int(w.doc_tokens_mean),
        "k": w.k,
        "stages": w.n_stages,
        "block_tokens": w.block_tokens,
        "gpu_tier_tokens": w.gpu_capacity_tokens,
        "host_tier_tokens": w.host_capacity_tokens,
        "parallelism": f"dp{world} (tree replicas) + corpus shards",
        "l2": (f"inputs larger than L2 (corpus shard scan {shard_rows * 768 * 2 / 1e6:.0f} MB, "
               f"KV pages {w.model.kv_bytes_per_token * int(w.doc_tokens_mean) * w.k / 1e6:.0f} "
               f"MB of cached documents per request)"),
    }


def cpu_baseline(args, w, R, steps, sizes, profile, profile_src) -> dict:
    """The reference CPU path (oracle/ref_path.py) on a bounded sample: 2 timed steps of 2
    requests each, plus ragsim's host decision time per request (1 core) and a CPU
    KV-gather GB/s comparator."""
    from oracle import ref_path

    res = ref_path.run_cpu_path(w, steps, sizes, profile, R=R, n_warm=args.cache_warm_steps,
                                n_steps=2, n_sample=2)
    block_bytes = w.block_tokens * w.model.kv_bytes_per_token
    return {"value": round(res["value"], 4), "unit": "req/s", "cores": res["cores"],
            "kind": "port", "sample": res["sample"] + f"; {res['steps']} timed steps",
            "doc_hit_rate": res["doc_hit_rate"],
            "host_decision": ref_path.host_decision_us(
                w, os.path.join(ROOT, profile_src) if profile_src.endswith(".csv") else None),
            "kv_gather": ref_path.cpu_gather_gbs(block_bytes, n_blocks=max(32, int(2e9 // block_bytes)),
                                                 n_pick=min(32, max(4, int(1e9 // block_bytes))))}


def run_reference(args, dist: Dist):
    """--impl reference: the reference's CPU path on the host cores (oracle/ref_path.py):
    ragsim's unmodified KnowledgeTree decisions + the oracle port of the three kernels,
    each step a bounded sample of the GPU arm's step, every timed second measured.
    Under torchrun only rank 0 runs."""
    if dist.world > 1 and dist.rank != 0:
        return
    from oracle import ref_path

    one = Dist()
    w, R, steps, sizes, _ = build_workload(args, one)
    profile, profile_src = tree_profile(w)
    W, K = args.warmup, args.steps
    res = ref_path.run_cpu_path(w, steps, sizes, profile, R=R, n_warm=args.cache_warm_steps + W,
                                n_steps=K, n_sample=args.ref_sample)
    value = res["value"]
    cpu = {"value": round(value, 4), "unit": "req/s", "cores": res["cores"], "kind": "port",
           "sample": res["sample"]}
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": "req/s",
        "n_gpus": dist.world, "steps": res["steps"], "warmup": W,
        "ms_per_step": round(res["ms_per_step"], 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": bench_config(w, R, dist.world),
        "doc_hit_rate": res["doc_hit_rate"],
        "retrieval_final_stage_matches_ground_truth": res["retrieval_matches_ground_truth"],
        "tree_profile": profile_src,
        "cpu_baseline": cpu,
        "e2e": {"value": round(value, 4), "unit": "req/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "warmup_note": (f"{args.cache_warm_steps} cache-warm + {W} warmup steps replayed "
                        f"untimed on the tree (decisions only)"),
    }))


def main():
    args = parse()
    dist = Dist()
    if args.impl == "reference":
        run_reference(args, dist)
        return
    res = run_ours(args, dist, emit=False)
    if (res is not None and dist.world == 1 and not args.no_ttft and not args.no_hit_sweep
            and args.workload + "-qpool" in WORKLOAD_NAMES()):
        res["hotpath_vs_hit_rate"] = guarded(hit_rate_sweep, args, dist)
    if res is not None:
        print(json.dumps(res))
    if dist.pg is not None:
        dist.pg.destroy_process_group()


if __name__ == "__main__":
    main()
