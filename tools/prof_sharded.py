"""A few steps of a sharded integrator at world size 1 (ncu launch-list target).
usage: prof_sharded.py config steps exchange   (config: bru_etd | bru_l2b | nls_ee | nls_etd;
exchange: nccl | kpnccl | peer)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist

import paper_2304_02327_b200 as kp
from paper_2304_02327_b200 import parallel, problems
from paper_2304_02327_b200.integrators import _upload_factors

name, steps, exch = sys.argv[1], int(sys.argv[2]), sys.argv[3]
os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29573")
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
be = parallel.CudaBackend(0)
comm = {"nccl": lambda: parallel.Comm(), "kpnccl": lambda: parallel.NcclComm(be),
        "peer": lambda: parallel.PeerComm(be)}[exch]()
builder, method = {"bru_etd": ("brusselator", "etd2rk"), "bru_l2b": ("brusselator", "lawson2b"),
                   "nls_ee": ("nls", "exp_euler"), "nls_etd": ("nls", "etd2rk")}[name]
c = getattr(problems, builder)(method=method)
ud = kp.to_device(c.u0)
flat = ud.permute(*reversed(range(ud.ndim))).reshape(-1)
K = _upload_factors(c.K)
it = parallel.make_sharded_integrator(kp, be, comm, method, list(c.u0.shape), K, c.g, 0.0,
                                      c.t_final * steps / c.n_steps, steps)
try:
    it.run(flat, steps)
except kp.DivergenceError:
    pass
torch.cuda.synchronize()
print("ok", name, steps, exch)
dist.destroy_process_group()
