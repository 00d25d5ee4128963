"""Per-layer / per-component device-vs-oracle error report (debug aid)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import mglp_oracle as O  # noqa: E402
from paper_2601_09026_b200 import LayerStack, StackConfig, State, serial_forward  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


name = sys.argv[1] if len(sys.argv) > 1 else "enc_small"
g = np.load(os.path.join(ROOT, "tests", "golden", name + ".npz"))
m = json.loads(str(g["meta"]))
sc = StackConfig(kind=m["kind"], d=m["d"], heads=m["heads"], ffn=m["ffn"], n_enc=m["n_enc"],
                 n_dec=m["n_dec"], buffer_open=m["buffer_open"], buffer_close=m["buffer_close"])
st = LayerStack(sc, m["seed"])
st.set_params(g["params"])
ost = O.Stack(O.StackConfig(kind=m["kind"], d=m["d"], heads=m["heads"], ffn=m["ffn"],
                            n_enc=m["n_enc"], n_dec=m["n_dec"], buffer_open=m["buffer_open"],
                            buffer_close=m["buffer_close"]), g["params"])
B, sx, sy, d = m["B"], m["sx"], m["sy"], m["d"]
z = State.from_flat(g["z0"], B, sx, sy, d)
lam = State.from_flat(g["lamN"], B, sx, sy, d)
oz = O.State.from_flat(g["z0"], B, sx, sy, d)
ol = O.State.from_flat(g["lamN"], B, sx, sy, d)
comps = O.layer_components(False, d, m["ffn"])
for layer in range(min(3, st.total_layers())):
    s_dev = st.step(layer, 0.37, z).flat()
    s_ref = ost.step(layer, 0.37, oz).flat()
    r_dev = st.adjoint_step(layer, 0.37, z, lam).flat()
    r_ref = ost.adjoint_step(layer, 0.37, oz, ol, None, 0.0).flat()
    gr = st.zero_grads()
    st.adjoint_step(layer, 0.37, z, lam, gr, 0.5)
    og = ost.zero_grads()
    ost.adjoint_step(layer, 0.37, oz, ol, og, 0.5)
    wg = O.Stack.flatten(og)
    print(f"layer {layer}: step {rel(s_dev, s_ref):.2e} adj {rel(r_dev, r_ref):.2e}")
    # per component of this layer's grads
    off = 0
    for L in range(layer):
        off += sum(int(np.prod(s)) for _, s in O.layer_components(ost.is_decoder(L), d, m["ffn"]))
    for cname, shp in O.layer_components(ost.is_decoder(layer), d, m["ffn"]):
        n = int(np.prod(shp))
        print(f"   {cname:12s} {rel(gr[off:off+n], wg[off:off+n]):.2e}  |ref| {np.abs(wg[off:off+n]).max():.2e}")
        off += n
traj = serial_forward(st, z)
otraj = O.serial_forward(ost, oz)
for i, (a, b) in enumerate(zip(traj, otraj)):
    print(f"serial point {i}: {rel(a.flat(), b.flat()):.2e}")
