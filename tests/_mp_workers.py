"""Worker processes of the multi-process GPU tests (not collected: no test_
prefix).  Each worker is one rank of a torch.distributed group on the single
B200 of the test box; the exchange goes through gloo (host staging), so no
rank's kernel ever waits on another rank's kernel: the ranks run the real
sharded device engine (slab images, row gathers, Gram closure, norm merge)
concurrently, and the collectives are real cross-process ones."""

import os

import numpy as np


def sharded_fit_worker(rank, world, port, x, R, cfg_kw, out_dir, synth_args=None):
    """distributed_fit on this rank: of the host tensor ``x`` (every rank
    slices its slabs), or, with ``synth_args`` = (dims, R, snr_db, seed,
    dtype), of a ShardedTensor whose three slabs this rank generates on the
    device.  Rank results go to out_dir/rank<r>.npz."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    os.environ["NTF_B200_SHARDED_GRAPH"] = "0"  # gloo collectives cannot be graph-captured
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1409_2383_b200 as P
        from paper_1409_2383_b200 import synth
        from paper_1409_2383_b200.distributed import PartitionPlan, ShardedTensor

        cfg = P.SolverConfig(**cfg_kw)
        if synth_args is None:
            res = P.distributed_fit(x, R, None, cfg, plan=world)
        else:
            dims, rr, snr, seed, dtype = synth_args
            spec = synth.SynthSpec.make(dims, rr, snr, seed)
            plan = PartitionPlan.uniform(dims, world)
            slabs = [synth.generate_box(spec, lo, hi, dtype=dtype)
                     for lo, hi in ShardedTensor.slab_boxes(dims, plan, rank)]
            res = P.distributed_fit(ShardedTensor(dims, plan, rank, slabs), R, None, cfg)
        out = dict(rfe=res.rfe, iterations=res.iterations)
        for m, f in enumerate(res.model.factors):
            out[f"factor{m}"] = np.asarray(f)
        if res.factor_history:
            for m in range(3):
                out[f"hist{m}"] = np.stack([np.asarray(it[m]) for it in res.factor_history])
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), **out)
    finally:
        dist.destroy_process_group()
