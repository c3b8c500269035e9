"""GPU: the library's NCCL communicator (rs_comm_*), the rollout path's one collective -- the
drafter-gradient all-reduce of the prompt-sharded KD update (learner.cpp:68-80).

A gpurun box has one GPU, so the communicator runs with one rank here (NCCL refuses two ranks on
one device): ids, creation, the in-place device all-reduce on a library-owned gradient buffer
and the host reductions must be exact identities, and the distributed KD step through the
communicator must equal the plain kd_update. The rendezvous and the rank arithmetic are covered
with two processes on CPU (tests/test_multiproc.py)."""
import pytest
import torch

import paper_2510_26475_b200 as rb
from paper_2510_26475_b200.distributed import Comm, kd_step_distributed_transformer

pytestmark = pytest.mark.gpu


def test_single_rank_comm_is_identity():
    assert Comm.nccl_version() >= 21800
    c = Comm(1, 0, Comm.unique_id())
    assert (c.size, c.rank) == (1, 0)
    buf = rb.DeviceBuffer.floats(1 << 20)
    host = torch.arange(1 << 20, dtype=torch.float32).numpy()  # kept alive across the copy
    rb._check(rb.lib().rs_memcpy_h2d(buf.device.handle, rb.ctypes.c_void_p(buf.ptr),
                                      rb.ctypes.c_void_p(host.ctypes.data), buf.nbytes))
    before = buf.to_numpy().copy()
    c.allreduce_(buf)
    buf.device.sync()
    assert (buf.to_numpy() == before).all()
    assert c.allreduce_host([1.5, -2.0, 7.0]) == [1.5, -2.0, 7.0]
    assert c.allreduce_host([3.0], "max") == [3.0]
    c.barrier()
    with pytest.raises(rb.InvalidArgument):
        c.allreduce_host([0.0] * 65)
    c.close()


def test_distributed_kd_step_through_comm_equals_kd_update():
    import random
    shape = rb.TransformerShape.tiny(vocab=512, max_ctx=128)
    tgt = rb.TransformerModel(shape, seed=41)
    drf = rb.EagleDrafter(tgt, seed=42, version=2)
    rng = random.Random(3)
    ss = [rb.RolloutSample([rng.randrange(511) for _ in range(4 + i)], [rng.randrange(512) for _ in range(5 + 2 * i)], [],
                           eos_bias=-1.0, reward=rng.random()) for i in range(4)]
    pol = rb.KDPolicy(interval=1, mode=0, lr=0.25)
    c = Comm(1, 0, Comm.unique_id())
    st = kd_step_distributed_transformer(drf, [s.reward for s in ss], [len(s.response) for s in ss], ss,
                                         list(range(len(ss))), pol, rb.SelectionRng(9), 0.01, comm=c)
    ref = rb.kd_update(drf, ss, pol, rb.SelectionRng(9), 0.01)
    assert st.loss == pytest.approx(ref.loss, rel=1e-12)
    for name in rb.EagleDrafter.GRAD_TENSORS:
        assert torch.equal(st.drafter.to_torch(name), ref.drafter.to_torch(name)), name
