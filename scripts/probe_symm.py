import os, torch, torch.distributed as dist
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29555", RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
import torch.distributed._symmetric_memory as symm
print("torch", torch.__version__)
try:
    print("has_multicast_support", symm.has_multicast_support("cuda", 0) if hasattr(symm, "has_multicast_support") else torch._C._distributed_c10d._SymmetricMemory.has_multicast_support(torch._C._distributed_c10d.DeviceType.CUDA, 0))
except Exception as e:
    print("has_multicast_support err", e)
try:
    t = symm.empty(1024, dtype=torch.float64, device="cuda")
    h = symm.rendezvous(t, dist.group.WORLD.group_name)
    print("handle", type(h), [a for a in dir(h) if not a.startswith('_')])
    print("multicast_ptr", getattr(h, "multicast_ptr", None))
    print("buffer_ptrs", getattr(h, "buffer_ptrs", None))
except Exception as e:
    import traceback; traceback.print_exc()
dist.destroy_process_group()
