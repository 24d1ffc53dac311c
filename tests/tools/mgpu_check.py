"""Multi-GPU parity check (run under torchrun, one process per GPU):
sharded replay of Task Bench graphs with P2P cross-shard edges, tokens
gathered to rank 0 and compared bit-exactly with the sequential oracle."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2508_16522_b200 import _native as N  # noqa: E402
from paper_2508_16522_b200.shard import ShardedGraph, lowering_stats  # noqa: E402
from paper_2508_16522_b200.taskbench import generate_graph  # noqa: E402


def main():
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, ws = dist.get_rank(), dist.get_world_size()
    cases = [("stencil_1d", 64 * ws, 50, 0, 0), ("nearest", 96 * ws, 20, 2, 3), ("fft", 128 * ws, 30, 0, 0),
             ("all_to_all", 32 * ws, 5, 0, 0), ("all_to_all", 300 * ws, 4, 0, 0), ("tree", 64 * ws, 12, 0, 0), ("stencil_1d", 1024 * ws, 200, 0, 0)]
    ok = True
    for pat, W, T, kind, arg in cases:
        g = generate_graph(pat, W, T, n_workers=min(W, 512 * ws), mapping="block", kind=kind, arg=arg)
        sg = ShardedGraph(g, ws, rank, local)
        for rep in range(3):
            sg.dev.run(seed=7 + rep, flags=N.TD_F_TALLY | N.TD_F_STATS)
            tok = sg.dev.tokens()
            tally = sg.dev.tally()
            mine = sg.local_nodes()
            parts = [None] * ws
            dist.all_gather_object(parts, (mine, tok[mine], tally[mine]))
            st = sg.dev.stats()
            if rank == 0:
                from oracle import seq
                full = np.zeros(g.n, np.uint64)
                tl = np.zeros(g.n, np.uint32)
                for m, t, c in parts:
                    full[m] = t
                    tl[m] = c
                want = seq.run_c(g.n, g.pred.ptr, g.pred.iv, g.kind, g.arg, seed=7 + rep)
                good = np.array_equal(full, want) and (tl == 1).all()
                ls = lowering_stats(g, sg.node_rank)
                print(f"{pat} W={W} T={T} rep={rep}: parity={good} cross_rank_edges(rank0)={st['cross_rank_edges']} "
                      f"ext_pairs={ls['ext_pairs']}", flush=True)
                ok &= good
        dist.barrier()
        sg.dev.close()
    # config-5 mini-app sharded by blocks of tiles: halo rows of other shards
    # are read from the peer's grid over NVLink
    from paper_2508_16522_b200.taskbench import generate_stencil2d
    for nx, ny, T, mapping in [(512, 512, 4, "block"), (1024, 2048, 5, "block"), (1024, 2048, 5, "shard_cyclic"), (1024, 2048, 5, "shard_block")]:
        g = generate_stencil2d(nx, ny, T, n_workers=min((nx // 64) * (ny // 64), 256 * ws), mapping=mapping,
                               shards=ws)
        sg = ShardedGraph(g, ws, rank, local, stencil2d=(nx, ny))
        for rep in range(2):
            sg.dev.run(seed=3 + rep, flags=N.TD_F_TALLY)
            mine = sg.local_nodes()
            tok = sg.dev.tokens()
            grid = sg.dev.stencil2d_grid((T - 1) & 1)
            parts = [None] * ws
            dist.all_gather_object(parts, (mine, tok[mine], grid))
            if rank == 0:
                from oracle import seq
                want_tok, want_grid = seq.stencil2d_tokens(g, seed=3 + rep)
                full = np.zeros(g.n, np.uint64)
                fgrid = np.zeros_like(want_grid)
                nt = (nx // 64) * (ny // 64)
                for r, (m, t, gr) in enumerate(parts):
                    full[m] = t
                    # each shard owns whole tiles: copy its tiles from its grid
                    tiles = np.unique(m % nt)
                    for tile in tiles:
                        ty, tx = divmod(int(tile), nx // 64)
                        fgrid[ty * 64:(ty + 1) * 64, tx * 64:(tx + 1) * 64] = gr[ty * 64:(ty + 1) * 64, tx * 64:(tx + 1) * 64]
                good = np.array_equal(full, want_tok) and np.array_equal(fgrid, want_grid)
                print(f"stencil2d {nx}x{ny} T={T} {mapping} rep={rep}: parity={good}", flush=True)
                ok &= good
        dist.barrier()
        sg.dev.close()
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    sys.exit(0 if flag.item() else 1)


if __name__ == "__main__":
    main()
