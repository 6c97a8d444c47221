"""One rank of tests/test_gpu_multiprocess.py (run as a subprocess): block
RANK of make_blocks_for_consensus on cuda:0, joined to the other rank by a
torch.distributed gloo group through libbsgpu's host communicator; runs one
consensus round with the product's pack / unpack / residual kernels and
writes the block's results as JSON. Test infrastructure only."""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
sys.path.insert(0, HERE)


def main():
    import torch
    import torch.distributed as dist

    from paper_2405_13943_b200 import api
    from test_gpu_train import make_blocks_for_consensus, setup_device_block

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    relax, fd = os.environ["RELAX"] == "1", int(os.environ["FD"])
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a, b, shared, zprev = make_blocks_for_consensus(fd=fd)
    dev = setup_device_block((a, b)[rank], shared, rank, zprev, api.penalties())
    calls = []

    def allreduce(arr, op):
        t = torch.from_numpy(arr)  # shares the pinned staging buffer
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        calls.append((len(arr), str(arr.dtype), op))

    dev.comm_init_host(allreduce, world, rank)
    dev.set_round_timeout(60.0)
    res = dev.consensus_round(1.6, relax, diagnostics=True)
    out = dict(res=res, z=dev.consensus().tolist(), duals=dev.duals().tolist(), anchor=dev.anchor().tolist(),
               calls=calls)
    with open(os.environ["OUT"], "w") as f:
        json.dump(out, f)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
