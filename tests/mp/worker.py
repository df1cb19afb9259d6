"""One rank of tests/test_gpu_multiproc.py (launched by torch.distributed.run, one process per
GPU, NCCL): the row-sharded solve through the public API; writes this rank's rows of Theta^K,
the gathered y and its rows of Xi, and the diagnostics of cr_primal to <out>/rank<r>.npz.

    worker.py <config> <N> <K> <p2p 0|1> <out_dir>
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import crdata  # noqa: E402
import paper_1608_02227_b200 as crp  # noqa: E402


def main():
    cfg_name, N, K, p2p, out = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), sys.argv[4] == "1", sys.argv[5]
    L = float(sys.argv[6])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = crdata.CONFIGS[cfg_name]
    X, ybar = crdata.make_problem(cfg, N=N)
    s = crp.Solver(X, ybar, cfg.gamma, L=L, prec=cfg.prec, group=dist.group.WORLD, p2p=p2p)
    s.solve(K)
    T = s.get_theta()[0]
    y, xi, st = s.primal()
    np.savez(os.path.join(out, f"rank{dist.get_rank()}.npz"), row0=s.row0, rows=s.rows, T=T, y=y, xi=xi,
             **{k: v for k, v in st.items()})
    s.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
