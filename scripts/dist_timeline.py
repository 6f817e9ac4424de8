"""Host-side timeline of the N-GPU set-up (torchrun): wall time of afsai_setup and
its stats, several repetitions (the first includes NCCL connection set-up)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
import afsai_inputs as ai
from paper_2010_14175_b200.api import Context, DeviceCSR, Factor
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
nx = 100
A = ai.poisson3d(nx, nx, nx * world)
n_loc = nx ** 3
dA = DeviceCSR.from_numpy(A, row_begin=rank * n_loc, n_rows=n_loc)
ctx = Context()
out = []
for r in range(4):
    torch.cuda.synchronize(); dist.barrier()
    t0 = time.perf_counter()
    F = Factor(ctx, dA, 20, 2, 0.0, 1000)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    st = F.stats()
    out.append({"wall_ms": (t1 - t0) * 1e3, **{k: st[k] for k in ["ms_total", "ms_rows", "ms_assemble", "ms_transpose", "ms_halo", "halo_rows"]}})
    F.close()
allr = [None] * world
dist.all_gather_object(allr, out)
if rank == 0:
    print(json.dumps(allr, indent=1))
dist.destroy_process_group()
