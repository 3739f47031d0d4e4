"""One-GPU emulation of rank 0's step of a P-rank c5 job: the native trevc_z_dist path
with MSTRSM_DIST_EMULATE_P=P and MSTRSM_DIST_TEST_UNPACK=1 runs rank 0's column shard, streams T's
panels through the broadcast buffer and unpacks them on the comm stream under the solve (the
receive-side copies a non-root rank does), gathers the P-rank triangular layout (the other ranks'
bytes as a device-to-device copy of the same volume) and unpacks all m columns.  NVLink transfer
time itself is not emulated (it is modelled in DESIGN §9).  Prints one JSON line per measurement.

    python tools/exp_dist_emul.py [P] [m]"""
import json
import os
import sys

P = int(sys.argv[1]) if len(sys.argv) > 1 else 8
os.environ["MSTRSM_DIST_EMULATE_P"] = str(P)
os.environ["MSTRSM_DIST_TEST_UNPACK"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import paper_1607_01477_b200 as ms  # noqa: E402
from paper_1607_01477_b200 import dist, inputs  # noqa: E402


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(e0.elapsed_time(e1))
    return min(out), sum(out) / len(out)


def main():
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
    ms.load()
    T = torch.from_numpy(inputs.c5_grcar_like(m)).cuda()
    cols = dist.shard_cols(m, P, 0, 16)
    best, mean = timed(lambda: ms.trevc(T, nb=128, cols=cols))
    print(json.dumps({"what": f"rank 0's shard solve alone (P = {P})", "ms_min": best, "ms_mean": mean}), flush=True)
    ms.comm_init(1, 0)
    best, mean = timed(lambda: ms.trevc_dist(T, m, nb=128))
    print(json.dumps({"what": f"emulated rank-0 step (P = {P}): streamed-panel receive copies under the solve, "
                              f"status all-reduce, P-rank gather volume (D2D stand-in), unpack",
                      "ms_min": best, "ms_mean": mean}), flush=True)
    ms.comm_destroy()
    best, mean = timed(lambda: ms.trevc(T, nb=128), reps=2)
    print(json.dumps({"what": "N = 1 TriangEig (all columns)", "ms_min": best, "ms_mean": mean}), flush=True)


if __name__ == "__main__":
    main()
