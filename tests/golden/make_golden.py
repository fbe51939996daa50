"""Regenerates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists and oracle/_ref is
built):  python tests/golden/make_golden.py
The fixtures pin the plain-C oracle restatement and the product's host code
even where oracle/_ref is unavailable.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, os.path.dirname(HERE))

from oracle import ref  # noqa: E402
import cases  # noqa: E402

SMALL = (16, 2, 4, 5.0, 3)  # ModelConfig small enough for compact fixtures


def main():
    R = ref()
    out = {}
    rng = np.random.default_rng(0)
    # neighbour lists: SPEC examples + random systems
    nl = cases.pack(cases.edge_systems(rng))
    ap = nl["atom_ptr"]
    for s in range(len(ap) - 1):
        i, j, d, u = R.neighbor_list(nl["pos"][ap[s]:ap[s + 1]], nl["Z"][ap[s]:ap[s + 1]], 5.0)
        out[f"nl{s}_i"], out[f"nl{s}_j"], out[f"nl{s}_d"], out[f"nl{s}_u"] = i, j, d, u
    for k, v in nl.items():
        out["nlbatch_" + k] = v
    # model: forward/backward/loss on generated molecules with the small config
    b = cases.with_heads(R.synth_generate(6, 42, mode=8, sigma=0.5, min_atoms=2, max_atoms=14,
                                          elements=cases.ORGANIC), SMALL[4], seed=2)
    b["energy_mask"][1] = 0
    b["force_mask"][2] = 0
    p = R.init_params(SMALL, 7)
    e, f = R.forward(SMALL, p, b)
    bd, ge, gf = R.loss_grad(b, SMALL[4], e, f)
    g = R.backward(SMALL, p, b, ge, gf)
    for k, v in b.items():
        out["mol_" + k] = v
    out.update(params=p, energy=e, forces=f, loss=np.array([bd["total"], bd["energy_term"], bd["force_term"]]),
               g_energy=ge, g_forces=gf, grads=g)
    # one train step with denoising + a reference table
    t = cases.random_table(SMALL[4], seed=3)
    mb = cases.mixed_batch(R, D=SMALL[4], seed=4, count=6)
    st = R.train_step(SMALL, 2, 3, mb, t, p, np.zeros_like(p), seed=11, step=2, clip=0.05)
    for k, v in mb.items():
        out["mix_" + k] = v
    for k, v in t.items():
        out["table_" + k] = v
    out.update(step_params=st["params"], step_v=st["rms_v"], step_loss=np.array([st["loss"], st["grad_norm"]]),
               step_grads=st["grads"])
    # scheduler / trace / rng
    tr = R.make_trace("lognormal", 5000, 2, 2000, mode=20, sigma=1.0, seed=3)
    out["trace"] = tr
    for mode in ("balanced", "greedy_only", "naive"):
        pl = R.plan(tr, 4, 2, 50, 9, mode)
        for k in ("sample", "worker", "atoms", "split", "chunk_rank", "worker_atoms"):
            out[f"plan_{mode}_{k}"] = pl[k]
        out[f"plan_{mode}_stats"] = np.array([pl["n_batches"], pl["dropped"], pl["max_imbalance"],
                                              pl["mean_imbalance"], pl["monotonicity_violations"],
                                              pl["growth_events"]], np.float64)
    out["normals"] = R.rng_normals(123, 257)
    out["perm"] = R.rng_permutation(5, 100)
    out["denoise_noisy"], out["denoise_labels"] = R.apply_noise(b["pos"][:5], b["Z"][:5], 0.3, 1, 99)
    np.savez_compressed(os.path.join(HERE, "reference_v1.npz"), **out)
    print("wrote", os.path.join(HERE, "reference_v1.npz"), len(out), "arrays")


if __name__ == "__main__":
    main()
