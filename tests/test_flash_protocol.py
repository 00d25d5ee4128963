"""CPU checks of the mbarrier protocols of the warp-specialised attention
kernels (attn_flash.cu) through their randomised simulators: random TMA and
tensor-pipe latencies and warp speeds, every parity wait checked for the phase
it means, every shared-memory stage / K, V tile / TMEM buffer / accumulator
checked for use-after-overwrite. The simulators must also catch a seeded
protocol bug, so a green run is evidence rather than a vacuous pass."""
import importlib.util
import os
import types

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(name):
    spec = importlib.util.spec_from_file_location(name, os.path.join(ROOT, "tools", name + ".py"))
    m = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(m)
    return m


def test_kv_backward_protocol_random_schedules():
    sim = _load("flash_kv_protocol_sim")
    steps = sum(sim.simulate(seed) for seed in range(300))
    assert steps > 1000


@pytest.mark.parametrize("bug,fragment", [
    (("if klast >= 0:\n                        while", "if False:\n                        while"), "K/V overwritten"),
    (("while bar_state[kk] < NC:", "while False:"), "before every group read"),
    (('while not bM[kl % KST].ready(kl // KST, f"cmp{c} bM"):', "while False:"), "accumulator not complete"),
    (('while not bM[s].ready((k - KST) // KST, "tma bM")',
      'while not bM[s].ready(max(k - KST + 1, 0) // KST, "tma bM")'), ""),
])
def test_kv_protocol_simulator_catches_seeded_bugs(bug, fragment):
    src = open(os.path.join(ROOT, "tools", "flash_kv_protocol_sim.py")).read()
    assert bug[0] in src
    m = types.ModuleType("mutant")
    exec(compile(src.replace(*bug).replace('if __name__ == "__main__":', "if False:"), "mutant", "exec"),
         m.__dict__)
    for seed in range(400):
        try:
            m.simulate(seed)
        except AssertionError as e:
            assert fragment in str(e)
            return
    pytest.fail("seeded protocol bug not detected")


def test_forward_protocol_random_schedules():
    """the single-pass forward's protocol (tools/flash_protocol_sim.py)"""
    import random

    sim = _load("flash_protocol_sim")
    for seed in range(200):
        rng = random.Random(seed)
        probs = [rng.choice([1, 2, 3, 4, 5, 6, 8]) for _ in range(rng.randint(1, 4))]
        assert sim.run(seed, probs) is None, (seed, probs)
