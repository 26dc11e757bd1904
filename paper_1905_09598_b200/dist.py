"""Multi-GPU orchestration for libsom: plumbing only.

* Document sharding (batch mapping, QE, TE): rank r maps the contiguous
  documents ``shard_range(n, r, P)``; per-document outputs stay sharded and
  are identical to P = 1; the error sums (sum of sqrt(D1), count of
  non-adjacent BMU pairs, document count) are reduced with one all-reduce
  (NCCL on GPUs; gloo works for the CPU tests).
* Neuron sharding (online training of one large map): ``ShardedSOM`` puts
  each rank's handle in sharded mode (``som_comm_init``), exchanges the
  64-byte CUDA IPC handles of the per-rank mailboxes with an all-gather, and
  hands them to libsom (``som_comm_set_peers_ipc``).  The per-step exchange
  itself happens inside the training kernel (peer-memory stores over
  NVLink), not here.

Only ``torch.distributed`` calls live in this module; all arithmetic runs in
libsom's kernels.
"""
from __future__ import annotations

from . import som as _som


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced [lo, hi) of n items for rank (sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def neuron_owner(u: int, world: int) -> tuple[int, int]:
    """(rank, local index) of global unit u under the cyclic neuron sharding."""
    return u % world, u // world


def broadcast_unique_id(rank: int, group=None, make_id=None) -> bytes:
    """Rank 0 creates the 128-byte NCCL unique id (som_comm_unique_id) and
    every rank receives it over torch.distributed (any backend)."""
    import torch.distributed as dist

    make_id = make_id or _som.som_comm_unique_id
    obj = [make_id() if rank == 0 else None]
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


def init_nccl(h, rank: int, world: int, shard_mode: int, group=None) -> None:
    """Bind libsom's own NCCL communicator to handle h (som_comm_init_nccl):
    SOM_SHARD_DOCS makes som_errors / som_errors_csr reduce their fp64 sum
    and int64 counts over the ranks inside the library."""
    uid = broadcast_unique_id(rank, group)
    _som.som_comm_init_nccl(h, rank, world, uid, shard_mode)


def reduce_errors(qe_local: float, te_local: float, n_local: int, group=None, device=None) -> tuple[float, float]:
    """Host-side model of the document-sharded error reduction, used by the
    CPU (gloo) tests: QE = sum_r qe_r n_r / sum_r n_r (qe_r n_r is the rank's
    fp64 sum of sqrt(D1)); TE likewise from the integer counts.  On GPUs the
    library reduces the fp64 sums and int64 counts itself over NCCL
    (init_nccl with SOM_SHARD_DOCS); this function is not on that path."""
    import torch
    import torch.distributed as dist

    t = torch.tensor([qe_local * n_local, round(te_local * n_local), float(n_local)], dtype=torch.float64,
                     device=device)
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, group=group)
    s, bad, n = (float(v) for v in t.cpu())
    return s / n, bad / n


def errors_doc_sharded(m: "_som.SOM", X_shard, group=None, device=None) -> tuple[float, float]:
    """QE and TE of the whole (document-sharded) corpus.  The handle must be
    bound with init_nccl(..., SOM_SHARD_DOCS): som_errors then maps this
    rank's shard and reduces the fp64 sum and int64 counts over NCCL inside
    libsom (collective; an empty shard passes n = 0)."""
    n_local = int(X_shard.shape[0])
    return _som.som_errors(m.h, X_shard, n_local)


def exchange_handles(blob: bytes, group=None) -> list[bytes]:
    """All-gather one bytes object per rank (rank order)."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out: list = [None] * world
    dist.all_gather_object(out, blob, group=group)
    return out


class ShardedSOM:
    """A rows x cols map whose units are dealt cyclically over the ranks of
    `group`; one handle per rank on its own GPU."""

    def __init__(self, rows: int, cols: int, dim: int, topology: int, rank: int, world: int, device: int = 0,
                 group=None, peers_dev: list[int] | None = None, defer_peers: bool = False):
        self.rows, self.cols, self.dim, self.rank, self.world = rows, cols, dim, rank, world
        self.N = rows * cols
        self.group = group
        self.h = _som.som_create(rows, cols, dim, topology, device)
        _som.som_comm_init(self.h, rank, world)
        self.n_local = _som.som_comm_local_units(self.h)
        if defer_peers:
            pass                       # caller connects with set_peers(mailbox pointers)
        elif peers_dev is None and world > 1:
            handles = exchange_handles(_som.som_comm_mailbox_ipc(self.h), group)
            _som.som_comm_set_peers_ipc(self.h, handles)
        elif peers_dev is not None:
            _som.som_comm_set_peers_dev(self.h, peers_dev)

    def mailbox_ptr(self) -> int:
        return _som.som_comm_mailbox_ptr(self.h)

    def set_peers(self, mailboxes: list[int]) -> None:
        _som.som_comm_set_peers_dev(self.h, mailboxes)

    def close(self):
        if self.h:
            _som.som_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_weights(self, W_full) -> None:
        _som.som_set_weights(self.h, W_full)

    def get_local_rows(self, W_full) -> None:
        """Write this rank's rows (u = rank + world*l) into the full buffer."""
        _som.som_get_weights(self.h, W_full)

    def gather_weights(self, device=None):
        """Full N x dim map on every rank: own rows + all-reduce(SUM) of zeros elsewhere."""
        import torch
        import torch.distributed as dist

        W = torch.zeros(self.N, self.dim, dtype=torch.float32, device=device)
        _som.som_get_weights(self.h, W)
        if dist.is_initialized() and self.world > 1:
            dist.all_reduce(W, group=self.group)
        return W

    def train_online(self, X, n: int, epochs: int, alpha0: float, sigma0: float, seed: int, sched=None,
                     t_begin: int = 0, t_end: int = -1, bmu_log=None, barrier=None) -> None:
        """Collective: every rank calls with the same arguments.  `barrier`
        (default torch.distributed.barrier) separates consecutive calls."""
        if barrier is None:
            import torch.distributed as dist

            def barrier():
                if dist.is_initialized() and self.world > 1:
                    dist.barrier(group=self.group)
        barrier()
        _som.som_train_online(self.h, X, n, epochs, alpha0, sigma0, sched, seed, t_begin, t_end, bmu_log)
        barrier()


__all__ = ["shard_range", "neuron_owner", "broadcast_unique_id", "init_nccl", "reduce_errors", "errors_doc_sharded",
           "exchange_handles", "ShardedSOM"]
