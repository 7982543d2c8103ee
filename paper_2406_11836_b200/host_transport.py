"""Host-staged transport for the multi-rank step (dgs_host_transport): the
C-ABI's exchanges and loss all-reduce go through torch.distributed (gloo)
between processes that may share one GPU (NCCL refuses two ranks on one
device).  Used by the multi-rank tests and `bench.py --transport host`; the
production path is the context's NCCL communicator."""
import ctypes as C

import numpy as np
import torch
import torch.distributed as dist


class GlooTransport:
    def __init__(self):
        self.pending = []

    def send(self, user, buf, nbytes, peer):
        try:
            t = torch.from_numpy(np.ctypeslib.as_array((C.c_uint8 * nbytes).from_address(buf)).copy())
            self.pending.append((dist.isend(t, dst=int(peer)), t, None, 0))
            return 0
        except Exception:
            return 1

    def recv(self, user, buf, nbytes, peer):
        try:
            t = torch.empty(int(nbytes), dtype=torch.uint8)
            self.pending.append((dist.irecv(t, src=int(peer)), t, buf, int(nbytes)))
            return 0
        except Exception:
            return 1

    def flush(self, user):
        try:
            for work, _, _, _ in self.pending:
                work.wait()
            for _, t, buf, nbytes in self.pending:
                if buf is not None:
                    C.memmove(buf, t.numpy().ctypes.data, nbytes)
            self.pending = []
            return 0
        except Exception:
            return 1

    def allreduce(self, user, buf, n):
        try:
            arr = np.ctypeslib.as_array(buf, shape=(int(n),))
            t = torch.from_numpy(arr.copy())
            dist.all_reduce(t)
            arr[:] = t.numpy()
            return 0
        except Exception:
            return 1
