"""The reference CPU path of the bench (oracle/ref_path.py) and the headline step's decisions.

* The GPU arm's batched step (HotPath.admit_batch, then commit every admission) makes
  exactly the decisions ragsim's own unmodified KnowledgeTree makes under the same call
  sequence (PlainTreeReplay = SimulationEngine._admit/_commit, simulator.py:481-534):
  same alpha/beta/matched nodes per admission, same carry, same tree snapshot after
  every step (tree.py:514-527).
* `bench.py --impl reference` never loads libragcache_b200.so and times real work.
"""

import json
import os
import subprocess
import sys

import pytest

from paper_2404_12457_b200._ragsim import ragsim_available

pytestmark = pytest.mark.skipif(not ragsim_available(), reason="ragsim not importable")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name,n_steps,R,gpu,host", [
    ("tiny-1k", 40, 16, 6000, 16384),          # two tiers: swap-outs, swap-ins, host frees
    ("llama2-7b-top5", 12, 12, 40_000, 160_000),  # configs[2] tiers
])
def test_batched_step_decisions_equal_plain_reference_tree(name, n_steps, R, gpu, host):
    import dataclasses

    from oracle.ref_path import PlainTreeReplay, admit_step
    from paper_2404_12457_b200.hotpath import HotPath
    from paper_2404_12457_b200.pool import accounting_pool
    from paper_2404_12457_b200.workloads import WORKLOADS, make_stream, pool_blocks
    from ragsim.cost_model import synthetic_profile

    w = dataclasses.replace(WORKLOADS[name], gpu_capacity_tokens=gpu, host_capacity_tokens=host)
    trace, sizes = make_stream(w, n_steps * R)
    steps = [trace[i * R:(i + 1) * R] for i in range(n_steps)]
    prof = synthetic_profile()
    ng = pool_blocks(gpu, w.block_tokens, sizes.values(), R * (w.k + 1))
    nh = pool_blocks(host, w.block_tokens, sizes.values(), 0)
    hp = HotPath(w.model, gpu_capacity_tokens=gpu, host_capacity_tokens=host,
                 block_tokens=w.block_tokens, num_gpu_blocks=ng, num_host_blocks=nh, sizes=sizes,
                 profile=prof, pool=accounting_pool(ng, nh, w.block_tokens))
    plain = PlainTreeReplay(gpu, host, sizes, prof)
    carry_h, carry_p = [], []
    for batch in steps:
        bh = carry_h + list(batch)
        adm = hp.admit_batch([(r.id, r.doc_sequence, r.prompt_tokens) for r in bh[:R]])
        carry_h = bh[len(adm):]
        padm, carry_p = admit_step(lambda r: plain.admit(r.doc_sequence, r.prompt_tokens),
                                   carry_p + list(batch), R)
        assert [r.id for r, _ in padm] == [a.req_id for a in adm]
        assert [r.id for r in carry_p] == [r.id for r in carry_h]
        for a, (_, (matched, alpha, beta, moved)) in zip(adm, padm):
            assert (a.alpha, a.beta, a.swapped_in_tokens) == (alpha, beta, moved)
            assert [n.serial for n in a.matched] == [n.serial for n in matched]
        for a in adm:
            hp.commit(a)
        for r, a in padm:
            plain.commit(r.doc_sequence, a)
        assert hp.tree.snapshot() == plain.tree.snapshot()
    assert hp.tree.gpu.used == plain.tree.gpu.used and hp.tree.host.used == plain.tree.host.used


def test_reference_arm_runs_without_the_native_library():
    code = (
        "import json, sys; sys.argv = ['bench.py', '--impl', 'reference', '--workload', "
        "'tiny-1k', '--steps', '2', '--warmup', '1', '--cache-warm-steps', '3']\n"
        "import bench\n"
        "bench.main()\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'so_loaded': 'libragcache_b200' in maps}))\n"
    )
    res = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True, text=True,
                         timeout=600)
    assert res.returncode == 0, res.stderr[-3000:]
    lines = [json.loads(l) for l in res.stdout.splitlines() if l.startswith("{")]
    line, maps = lines[0], lines[-1]
    assert maps == {"so_loaded": False}
    assert line["impl"] == "reference" and line["value"] > 0 and line["steps"] == 2
    assert line["retrieval_final_stage_matches_ground_truth"]
    assert line["config"]["workload"] == "tiny-1k"
    assert line["ms_per_step"] * line["steps"] < 600_000
