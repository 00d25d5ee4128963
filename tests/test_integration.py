"""The drop-in, end to end: the reference's own
Trainer (proj/src/training.cpp, UNMODIFIED) compiled with its engine type
swapped for integration/mglp_cuda_engine.hpp's CudaLayerParallelEngine
(integration/Makefile, -include swap_engine.hpp) runs run_training with every
layer-parallel forward / backward on the B200 through the C-ABI; the stock
reference (oracle/_ref) runs the same configuration on the CPU. Metrics rows
(mode, budgets, losses, convergence factors), the switch decision and the
final MGLP v1 parameters must agree at the north-star 1e-4."""
import os
import subprocess

import numpy as np
import pytest

from oracle import ref as R
from paper_2601_09026_b200 import training as T
from paper_2601_09026_b200.controller import IndicatorConfig
from paper_2601_09026_b200.engine import SolveConfig, StackConfig

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "integration", "_build", "swap_trainer")
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not R.available() or not os.path.exists(BIN),
                                 reason="reference oracle / swap_trainer not built")]
KIND = {"encoder": 0, "decoder_only": 1, "encoder_decoder": 2}
TASK = {"copy_sequence": 0, "token_classification": 1, "tiny_translation": 2}
MODE = {"serial": 0, "layer_parallel": 1, "switching": 2}


def configure(kind="encoder", task="copy_sequence", mode="layer_parallel", epochs=2,
              dropout=0.0, **ind):
    n_enc, n_dec = {"encoder": (8, 0), "decoder_only": (0, 8), "encoder_decoder": (4, 4)}[kind]
    stack = StackConfig(kind=kind, d=32, heads=2, ffn=64, n_enc=n_enc, n_dec=n_dec,
                        dropout=dropout)
    tk = T.TaskSpec(kind=task, vocab=16, seq_len=8, train_size=16, val_size=8, seed=1)
    mc = T.ModelConfig(stack=stack, vocab=16, max_seq=8)
    tc = T.TrainConfig(mode=mode, solve=SolveConfig(coarsen=2, levels=2, fwd_iters=2,
                                                    bwd_iters=1),
                       batch_size=4, epochs=epochs, seed=7, val_every=2,
                       indicator=IndicatorConfig(**ind))
    return tk, mc, tc


def run_swapped(tmp_path, tk, mc, tc):
    s, ind = mc.stack, tc.indicator
    args = [KIND[s.kind], TASK[tk.kind], s.d, s.heads, s.ffn, s.n_enc, s.n_dec, tk.vocab,
            tk.seq_len, tk.train_size, tk.val_size, tc.batch_size, tc.epochs, MODE[tc.mode],
            tc.solve.coarsen, tc.solve.levels, tc.solve.fwd_iters, tc.solve.bwd_iters,
            ind.probe_period, repr(ind.threshold), ind.policy, ind.max_iter_cap,
            int(ind.use_probe_gradient), tc.val_every, repr(s.dropout)]
    out = str(tmp_path / "run")
    p = subprocess.run([BIN, out] + [str(a) for a in args], capture_output=True, text=True,
                       timeout=600)
    assert p.returncode == 0, p.stderr
    rd = lambda ext: open(out + ext, "rb").read()  # noqa: E731
    return dict(csv=rd(".csv").decode(), final_state=rd(".state"), switch=rd(".switch"),
                log=p.stdout)


def rows(csv):
    out = []
    for line in csv.strip().splitlines()[1:]:
        f = [x.strip() for x in line.split(",")]
        out.append(dict(batch=int(f[0]), loss=float(f[1]), val=float(f[2]), mode=f[3],
                        fi=int(f[4]), bi=int(f[5]), ff=float(f[6]), bf=float(f[7])))
    return out


def compare(dev, ref):
    dr, rr = rows(dev["csv"]), rows(ref["csv"])
    assert [(r["batch"], r["mode"], r["fi"], r["bi"]) for r in dr] == \
        [(r["batch"], r["mode"], r["fi"], r["bi"]) for r in rr]
    for d, r in zip(dr, rr):
        assert abs(d["loss"] - r["loss"]) <= 1e-4 * abs(r["loss"]), (d, r)
        assert abs(d["val"] - r["val"]) <= 2.0 / 32 + 1e-12
        for k in ("ff", "bf"):
            assert abs(d[k] - r[k]) <= 1e-4 * max(abs(r[k]), 1e-12), (k, d, r)
    dp = np.concatenate([t.ravel() for t in T.parse_checkpoint(dev["final_state"])["params"]])
    rp = np.concatenate([t.ravel() for t in T.parse_checkpoint(ref["final_state"])["params"]])
    assert np.abs(dp - rp).max() <= 1e-4 * np.abs(rp).max()


@pytest.mark.parametrize("args", [dict(),
                                  dict(kind="decoder_only"),
                                  dict(kind="encoder_decoder", task="tiny_translation"),
                                  dict(dropout=0.2)])
def test_reference_trainer_on_the_cuda_engine(tmp_path, args):
    tk, mc, tc = configure(**args)
    compare(run_swapped(tmp_path, tk, mc, tc), R.run_training(tk, mc, tc))


def test_reference_trainer_probes_and_switches_on_the_cuda_engine(tmp_path):
    """switching mode: ProbeScope doubles the budgets through config(), the
    measurement-only probe runs behind snapshot()/restore(), the monitor
    trips at threshold 1e-12 and the tail runs serial (test_training.cpp:151-174)"""
    tk, mc, tc = configure(mode="switching", probe_period=2, threshold=1e-12, policy=1,
                           use_probe_gradient=False)
    dev = run_swapped(tmp_path, tk, mc, tc)
    ref = R.run_training(tk, mc, tc)
    compare(dev, ref)
    assert dev["log"].split()[3] == str(ref["switch_batch"])
