"""Worker for test_gpu_multirank.test_p2p_ipc_two_processes (launched by torch.distributed.run):
each rank builds the same Simulation on cuda:0, exports its exchange buffers as CUDA IPC
handles, all-gathers the handles over gloo, maps the peer's, and runs three sharded steps.
With "stall" as the second argument only rank 0 steps (test_p2p_peer_timeout)."""
import os
import sys

import numpy as np
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1811_02761_b200 as g2  # noqa: E402
from paper_1811_02761_b200.gravitree import sample_model  # noqa: E402

out = sys.argv[1]
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
m, p, v = sample_model("m31", 100000, 5)
sim = g2.Simulation(g2.ParticleSystem(m, p, v), g2.GravParams(1.0, 2.0 ** -5, 2.0 ** -9),
                    g2.StepScheme(dt_max=1.0 / 64, adaptive=False))
sim.set_rebuild_every_step(True)
handles = [None] * world
dist.all_gather_object(handles, sim.p2p_export(rank, world))
sim.set_mesh_p2p(rank, world, handles)
sim.init()
if len(sys.argv) > 2 and sys.argv[2] == "stall":
    # rank 1 never steps: rank 0's exchange barrier must give up (G2_PEER_TIMEOUT_S) with a
    # ResourceError instead of spinning on the GPU forever
    if rank == 0:
        try:
            sim.step()
            outcome = "no error"
        except g2.ResourceError as e:
            outcome = "ResourceError: " + str(e)
        with open(os.path.join(out, "stall.txt"), "w") as f:
            f.write(outcome)
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0)
inter = 0
for _ in range(3):
    inter = sim.step().events.interactions
s = sim.system()
np.savez(os.path.join(out, f"rank{rank}.npz"), acc=s.acc, pos=s.pos, inter=inter)
dist.barrier()
dist.destroy_process_group()
