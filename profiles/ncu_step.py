"""Runs a few train steps of one workload for ncu: cfg2 (default), 'si' (4 x 1000-atom
Si supercells) or 'large' (bench.large_batch: 48 x 1000-atom supercells, > L2)."""
import sys, os, numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2505_22208_b200 as pk, cases, bench
cfg = pk.ModelConfig(**bench.CFG)
tc = pk.TrainConfig(seed=11)
which = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
if which == "si":
    parts = []
    for s in range(4):
        pos, Z, cell = cases.diamond_supercell(reps=5, seed=100 + s)
        n = len(Z)
        parts.append(dict(atom_ptr=np.array([0, n], np.int64), pos=pos, Z=Z, forces=np.zeros((n, 3)),
                          dataset_index=np.zeros(1, np.int32), energy_mask=np.ones(1, np.uint8),
                          force_mask=np.ones(1, np.uint8), energy=np.array([-4.6 * n]),
                          denoise=np.zeros(1, np.uint8), cell=cell[None]))
    batch = pk.concat(parts)
    table = None
elif which == "large":
    batch = bench.large_batch(pk)
    table = bench.fit_table(batch, bench.CFG["heads"])
else:
    pool, table, sched = bench.make_workload(pk, 1)
    from paper_2505_22208_b200.dist import shard
    batch = shard(pool, sched, 2, 0, 1, bench.BATCH_PER_GPU)
dev = pk.Device(cfg, seed=7)
if table is not None: dev.set_reference_table(table)
dev.stage(batch, tc, step=0, slot=0)
for _ in range(int(os.environ.get("NSTEPS", "3"))):
    r = dev.train_step_staged(0, sync=True)
print("N", r.n_atoms, "P", r.n_edges, "launches/step", dev.last_step_launches())
dev.close()
