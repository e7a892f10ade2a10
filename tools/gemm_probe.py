"""Skinny-GEMM probe for the model's dense projections (library GEMMs, not the hot path):
h[T, d_in] @ W for the Mistral-7B projections, W stored [d_in, d_out] (as model.py) vs
[d_out, d_in] (F.linear), CUDA-graph timed.  Prints achieved weight-read GB/s."""
import json
import sys

import torch

SHAPES = [(4096, 6144), (4096, 4096), (4096, 28672), (14336, 4096)]


def timed(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(reps):
                fn()
    torch.cuda.synchronize()
    g.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    for T in (1, 32, 64, 544):
        tot = {"nn": 0.0, "linear": 0.0}
        for din, dout in SHAPES:
            w = torch.randn(din, dout, device="cuda").to(torch.bfloat16)
            wt = w.t().contiguous()
            h = torch.randn(T, din, device="cuda").to(torch.bfloat16)
            a = timed(lambda: h @ w)
            b = timed(lambda: torch.nn.functional.linear(h, wt))
            tot["nn"] += a
            tot["linear"] += b
            gb = din * dout * 2 / 1e9
            print(json.dumps({"T": T, "din": din, "dout": dout, "nn_us": round(a * 1e3, 1),
                              "linear_us": round(b * 1e3, 1), "nn_gbs": round(gb / a * 1e3),
                              "linear_gbs": round(gb / b * 1e3)}), flush=True)
        print(json.dumps({"T": T, "layer_ms": {k: round(v, 4) for k, v in tot.items()},
                          "model_ms_32_layers": {k: round(32 * v, 3) for k, v in tot.items()}}))


if __name__ == "__main__":
    main()
