"""One configuration of tests/test_gpu_tc_rings.py in its own process (a protocol fault or hang
then cannot take the test session's CUDA context with it): the tcgen05 pass with the ring depths /
GEMM1 run-ahead given in the environment (CR_TC_STAGES, CR_TC_G1STAGES, CR_TC_G2STAGES,
CR_TC_G1_RUNAHEAD) and CR_TC_CHECK=1; prints a JSON line with the SHA-256 of Theta^K, the ring
depths cr_init chose and the check word.

    tc_ring_case.py <N> <n> <K> <L>
"""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import crdata  # noqa: E402
import paper_1608_02227_b200 as crp  # noqa: E402


def main():
    N, n, K, L = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
    X, ybar = crdata.random_problem(N, n, seed=N + n, fp32=True)
    s = crp.Solver(X, ybar, 1e-3, L=L, kernel="tc")
    s.solve(K)                       # CUDA-graph replays (fused reduce + prologue between passes)
    s.step()                         # and one eager step
    T = s.get_theta()[0]
    torch.cuda.synchronize()
    print(json.dumps({"sha": hashlib.sha256(np.ascontiguousarray(T).tobytes()).hexdigest(),
                      "check": s.tc_check_word, "kernel": s.kernel}), flush=True)
    s.close()


if __name__ == "__main__":
    main()
