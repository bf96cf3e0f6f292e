"""Host cost per call (wall clock, GPU work tiny so the host is the bottleneck):
ctypes no-op, current-stream lookup, and allreduce_average on registered / prepared
tensors with HVD_CFG_PROFILE off and on.  One JSON line per variant (us per call)."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1802_05799_b200 as hvd  # noqa: E402
from paper_1802_05799_b200 import _lib  # noqa: E402


def per_call(fn, n=3000):
    for _ in range(200):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    return (t1 - t0) / n * 1e6


def main():
    comm = hvd.init_virtual(1, 0, 64 << 20)
    x = [torch.randn(256, device="cuda")]
    reg = comm.register([x])
    prep = comm.prepare([x])
    lib = _lib.lib
    rows = [("ctypes hvd_rank", lambda: lib.hvd_rank(comm._h)),
            ("torch.cuda.current_stream", lambda: torch.cuda.current_stream().cuda_stream)]
    for prof in (0, 1):
        comm.set_config(_lib.HVD_CFG_PROFILE, prof)
        rows.append((f"allreduce_average registered profile={prof}", lambda: comm.allreduce_average(reg)))
        rows.append((f"allreduce_average prepared profile={prof}", lambda: comm.allreduce_average(prep)))
        rows.append((f"allreduce_average list profile={prof}", lambda: comm.allreduce_average([x])))
    for name, fn in rows:
        print(json.dumps({"variant": name, "us_per_call": per_call(fn)}), flush=True)
    comm.finalize()


if __name__ == "__main__":
    main()
