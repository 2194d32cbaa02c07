"""Host -> device upload of a C2-sized matrix through pinned staging chunks of
several sizes (engine._upload), timed with CUDA events around the whole call."""

import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2402_16712_b200 import engine  # noqa: E402


def run(n, m, chunk_doubles, reps=20):
    engine._STAGE_DOUBLES = chunk_doubles
    engine._STAGING.clear()
    X = np.random.default_rng(0).standard_normal((n, m))
    dev = torch.device("cuda", 0)
    for _ in range(3):
        engine._upload(X, dev)
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        d = engine._upload(X, dev)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t0)
    assert torch.equal(d.cpu(), torch.from_numpy(X))
    return np.median(ts) * 1e3


if __name__ == "__main__":
    print("threads", torch.get_num_threads())
    for n, m in [(2000, 2000), (10000, 10000)]:
        for mb in [1, 2, 4, 8, 16]:
            print(n, m, f"{mb} MB chunks: {run(n, m, mb << 17):.3f} ms")
    # the plain pageable copy and a pinned-whole copy, for scale
    X = np.random.default_rng(0).standard_normal((2000, 2000))
    t = torch.from_numpy(X)
    for _ in range(3):
        t.to("cuda")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        t.to("cuda")
    torch.cuda.synchronize()
    print("pageable .to(cuda):", (time.perf_counter() - t0) / 20 * 1e3, "ms")
    p = t.pin_memory()
    t0 = time.perf_counter()
    for _ in range(20):
        p.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    print("pinned DMA only:", (time.perf_counter() - t0) / 20 * 1e3, "ms")
    t0 = time.perf_counter()
    for _ in range(20):
        p.copy_(t)
    print("host copy into pinned:", (time.perf_counter() - t0) / 20 * 1e3, "ms")
