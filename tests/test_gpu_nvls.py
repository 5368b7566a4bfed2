"""C4 through the NVSwitch: the constraint-sharded solve with the flat
gradient buffer in symmetric memory and the in-switch multicast all-reduce (fsmt_mc_allreduce_f64)
must reproduce the NCCL constraint-sharded solve and the world-size-1 solve bit for bit (the
reduced values are on-grid integers, so the switch's fp64 adds are exact).  Needs >= 2 GPUs behind
NVSwitch with multicast support: skipped on the one-GPU boxes of this build (unmeasured there)."""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

KAPPAS = [0.5, 1.0, 2.0, 4.0, 8.0, 16.0]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _multicast_gpus() -> int:
    import torch
    if not torch.cuda.is_available():
        return 0
    n = torch.cuda.device_count()
    try:
        from torch._C._distributed_c10d import _SymmetricMemory, DeviceType
        if not _SymmetricMemory.has_multicast_support(DeviceType.CUDA, 0):
            return 0
    except Exception:
        return 0
    return n


def _worker(rank, world, port, nvls, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    import fsmt_gen
    import paper_2603_22877_b200 as P
    from paper_2603_22877_b200 import dist as D
    inst = fsmt_gen.config("cfg4s")
    s = P.Solver(rank)
    s.load_formula(inst.text)
    s.build_xbdd()
    s.set_params(kappas=KAPPAS, eta=0.05)
    d = s.get_dims()
    res = D.solve_constraint_sharded(s, d["n_bool"], d["n_real"], 64, 6, 21, KAPPAS, 1e-2, nvls=nvls)
    a, b = s.get_state()
    out[(nvls, world, rank)] = ((res.verdict, res.winner_restart, res.winner_stage, res.best_unsat, res.stages_run,
                                 res.x.tolist(), res.y.tolist()), (a.tolist(), b.tolist()))
    dist.destroy_process_group()


@pytest.mark.skipif(_multicast_gpus() < 2, reason="needs >= 2 GPUs with NVSwitch multicast (NVLS)")
def test_nvls_constraint_sharded_matches_nccl_and_world1():
    import torch.multiprocessing as mp
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(1, _port(), False, out), nprocs=1, join=True)
    mp.spawn(_worker, args=(2, _port(), False, out), nprocs=2, join=True)
    mp.spawn(_worker, args=(2, _port(), True, out), nprocs=2, join=True)
    ref = out[(False, 1, 0)]
    for rank in (0, 1):
        assert out[(False, 2, rank)] == ref
        assert out[(True, 2, rank)] == ref


def test_mc_allreduce_rejects_bad_arguments():
    """The entry point's argument checks run on any GPU (no multicast object needed)."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import fsmt_gen
    import paper_2603_22877_b200 as P
    s = P.Solver(0)
    s.load_formula(fsmt_gen.cfg1().text)
    s.build_xbdd()
    for args in ((0, 16, 0, 2), (1 << 20, 16, 2, 2), (1 << 20, 16, 0, 0)):
        with pytest.raises(P.FsmtError):
            s.mc_allreduce_f64(*args)
