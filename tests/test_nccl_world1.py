"""The sharded fit over a real NCCL process group on the one GPU a test box has
(world size 1: every collective of distributed.py -- the all-reduce(MIN) of the
upper bounds through l1b_fit_line's exchange hook, the all-gather of winner
records, the int64 all-reduce of the winners' bytes -- runs through NCCL on
CUDA tensors).  The multi-rank logic itself is covered with gloo, world 2 and 3,
in test_distributed.py."""

import numpy as np
import pytest
import torch
import torch.distributed as dist

import paper_2402_16712_b200 as l1b
from paper_2402_16712_b200.distributed import combine_winners, fit_lines_distributed, fit_subspace_distributed
from paper_2402_16712_b200.distributed import ub_exchange
from paper_2402_16712_b200.engine import PivotWinner

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def nccl_group():
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", store=dist.HashStore(), rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    assert dist.get_backend() == "nccl"
    yield
    dist.destroy_process_group()


def test_nccl_exchanges(nccl_group):
    ex = ub_exchange()
    assert ex(3.5) == 3.5
    assert np.array_equal(ex(np.array([1.0, -2.0, np.inf])), [1.0, -2.0, np.inf])
    v = np.array([-0.0, 1.5, -2.25, 5e-324])
    w = combine_winners([PivotWinner(3, 0.5, v, 1.0, 2.0, 2.0)], v.size)[0]
    assert w.pivot == 3 and w.v.tobytes() == v.tobytes() and (w.error, w.penalty_norm, w.objective) == (1.0, 2.0, 2.0)


def test_nccl_fit_lines_and_subspace_match_single_gpu(nccl_group):
    d, _ = l1b.gen_line_data(300, 2000, seed=4, noise_scale=1.0)
    X = np.array(d.values)
    lams = [1.0, 25.0, 400.0]
    got = fit_lines_distributed(X, lams)
    want = l1b.fit_lines(l1b.DataMatrix(X), lams)
    for a, b in zip(got, want):
        assert a.preserved == b.preserved and a.v.tobytes() == b.v.tobytes()
        assert (a.error, a.penalty_norm, a.objective) == (b.error, b.penalty_norm, b.objective)
    got = fit_subspace_distributed(X, 1.0, 2)
    want = l1b.fit_subspace(l1b.DataMatrix(X), 1.0, 2)
    for a, b in zip(got.components, want.components):
        assert a.preserved == b.preserved and a.v.tobytes() == b.v.tobytes() and a.objective == b.objective
