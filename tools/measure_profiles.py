"""Measure the B200 prefill profile T(alpha, beta) of each model shape and write it where the
bench tree and the acceptance re-runs read it: profiles/<shape>_b200_profile.csv (ragsim's
CSV format, cost_model.py:150-157), plus profiles/<shape>_b200_profile.json with the
measurement note and the one-token decode step at the configs' typical context.

    python tools/measure_profiles.py [shape ...]     (default: every BASELINE shape)
"""

import json
import os
import sys
import time

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2404_12457_b200.profile import decode_ms_per_token, measure_profile  # noqa: E402
from ragsim.cost_model import save_profile_csv  # noqa: E402

SHAPES = ("mistral-7b", "llama2-7b", "llama2-13b", "mixtral-8x7b")


def main():
    shapes = sys.argv[1:] or SHAPES
    out_dir = os.environ.get("OUT_DIR", os.path.join(ROOT, "profiles"))
    os.makedirs(out_dir, exist_ok=True)
    for shape in shapes:
        t0 = time.time()
        prof, info = measure_profile(shape, block_tokens=64, reps=3)
        info["seconds"] = round(time.time() - t0, 1)
        info["decode_ms_per_token"] = {str(c): round(decode_ms_per_token(prof, c), 4)
                                       for c in (544, 1056, 2592)}
        info["gpu"] = torch.cuda.get_device_name()
        save_profile_csv(prof, os.path.join(out_dir, f"{shape}_b200_profile.csv"))
        with open(os.path.join(out_dir, f"{shape}_b200_profile.json"), "w") as fp:
            json.dump(info, fp, indent=1)
        print(json.dumps({"shape": shape, **info}), flush=True)
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
