"""Exercise bench.py's N>1 C5 row-shard leg machinery on ONE GPU with world = 1: the child
process (own process group on a fresh port), shard setup (gen rows, IPC export/open with no
peers), one multi-step launch, readout_partial and the bitwise check against the unsharded
run. A one-rank "shard" waits on nothing, so nothing here waits on another kernel."""
import argparse
import json
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402

with socket.socket() as s:
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
os.environ.update(RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
args = argparse.Namespace(steps=20, warmup=3)
print(json.dumps(bench.c5_leg_in_children(args, 0, 1)))
dist.destroy_process_group()
