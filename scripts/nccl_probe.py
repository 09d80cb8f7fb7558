"""NVLink/NCCL probe: torch all_to_all_single and grouped send/recv bandwidth."""
import os, time, json
import torch, torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
res = {}
for mb in (8, 64, 256):
    n = mb * (1 << 20) // 4
    x = torch.ones(n * world, device=dev)
    y = torch.empty_like(x)
    for _ in range(3):
        dist.all_to_all_single(y, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        dist.all_to_all_single(y, x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    res[f"a2a_{mb}MB_per_peer_GBs_out"] = round(n * 4 * (world - 1) / (ms * 1e-3) / 1e9, 1)
if rank == 0:
    print(json.dumps(res))
dist.destroy_process_group()
