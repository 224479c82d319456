"""Multi-GPU semi-naive evaluation: hash-partitioned relations, per-iteration
exchange of new tuples.

One process per GPU (torch.distributed; NCCL over NVLink on a B200 box,
gloo for CPU-staged tests). Placement, decided once from the compiled plans:

* root keys are partitioned: rank r enumerates only root keys x with
  owner(x) == r (device: `srdl_root_own` zeroes the work of other keys), so
  the ranks' join outputs are disjoint and together complete;
* an index (relation, column order) whose every reader binds its leading
  column at the root is *partitioned* on that column (a rank stores only the
  rows it owns — exactly the rows its root keys need); any other index is
  *replicated*;
* delta indexes are only read by delta atoms, which are root-keyed: always
  partitioned;
* the identity index is the dedup authority. Partitioned: staged tuples go
  to the owner of their first column with one all-to-all and each rank
  computes the delta of its partition. Replicated: staged tuples are
  all-gathered and every rank computes the same global delta.

After compute-delta, each index receives its rows by one more all-to-all
(partitioned on another column) or all-gather (replicated), and an
all-reduce of the delta sizes decides termination (paper section 6
bulk-synchronous iterations; reference runtime.py:259-315 is the
single-process protocol this distributes).

owner(v) = ((v * 2654435761) mod 2^32 >> 8) mod world, identical in
csrc/setops.cu (`owner_of`) and `device.owner`.
"""

from __future__ import annotations

import torch

from . import device as dev
from .compiler import FULL

PART = "part"
REP = "rep"


def index_modes(compiled) -> dict:
    """{(relation, order): PART | REP} for the full indexes of a program, and
    {("delta", relation, order): REP} for delta indexes that some delta atom
    reads after constant columns (their leading column is not the root key,
    so they are kept complete)."""
    root_only: dict = {}
    modes = {}
    for stratum in compiled.strata:
        for plan in stratum.plans:
            for pa in plan.atoms:
                key = (pa.relation, tuple(pa.column_order))
                if pa.version != FULL:
                    if pa.n_const:
                        modes[("delta",) + key] = REP
                    continue
                root = pa.n_const == 0 and bool(pa.col_levels) and pa.col_levels[0] == 0
                root_only[key] = root_only.get(key, True) and root
    for name, orders in compiled.orders.items():
        for order in orders:
            modes[(name, tuple(order))] = PART if root_only.get((name, tuple(order)), True) else REP
    return modes


class DistContext:
    """Rank, world and the row-set collectives the fixpoint needs."""

    def __init__(self, group=None):
        import torch.distributed as td

        self.td = td
        self.group = group
        self.world = td.get_world_size(group)
        self.rank = td.get_rank(group)
        self.backend = str(td.get_backend(group))
        # gloo collectives run on host tensors (tests); NCCL on device memory
        self.staged = self.backend != "nccl"
        # payload this rank sent to other ranks (all-to-all rows, all-gather
        # rows), and the number of exchanges — DESIGN.md's per-iteration table
        self.sent_bytes = 0
        self.exchanges = 0

    def _dev(self):
        return torch.device("cpu") if self.staged else dev.device()

    def all_sum(self, value: int) -> int:
        t = torch.tensor([int(value)], dtype=torch.int64, device=self._dev())
        self.td.all_reduce(t, group=self.group)
        return int(t.item())

    def all_to_all_rows(self, rows: torch.Tensor, counts: list) -> torch.Tensor:
        """Send counts[r] consecutive rows (columns of `rows`) to rank r."""
        arity = rows.shape[0]
        cdev = self._dev()
        send_n = torch.tensor(counts, dtype=torch.int64, device=cdev)
        recv_n = torch.empty_like(send_n)
        self.td.all_to_all_single(recv_n, send_n, group=self.group)
        recv_counts = recv_n.tolist()
        send = rows.view(torch.int32).t().contiguous().to(cdev)  # (n, arity)
        recv = torch.empty((sum(recv_counts), arity), dtype=torch.int32, device=cdev)
        self.td.all_to_all_single(recv, send, recv_counts, list(counts), group=self.group)
        return recv.to(rows.device).t().contiguous().view(torch.uint32)

    def route(self, rows: torch.Tensor, key_col: int) -> torch.Tensor:
        """Rows delivered to the owner of their column key_col: one packing
        kernel writes the row-major send buffer grouped by owner and the
        per-rank counts on the device (srdl_route_pack), the counts are
        exchanged, ONE host read of (sent, received) counts sizes the
        receive buffer, one all-to-all moves the rows and srdl_unpack_rows
        restores the columns."""
        arity, n = rows.shape
        send, counts = dev.route_pack(rows, key_col, self.world)
        cdev = self._dev()
        counts_c = counts.to(cdev)
        recv_n = torch.empty_like(counts_c)
        self.td.all_to_all_single(recv_n, counts_c, group=self.group)
        both = torch.cat([counts_c, recv_n]).tolist()  # the exchange's one host read
        sent, got = both[:self.world], both[self.world:]
        recv = torch.empty(sum(got) * arity, dtype=torch.int32, device=cdev)
        self.td.all_to_all_single(recv, send.to(cdev), [g * arity for g in got], [c * arity for c in sent],
                                  group=self.group)
        self.sent_bytes += 4 * arity * (sum(sent) - sent[self.rank])
        self.exchanges += 1
        return dev.unpack_rows(recv.to(rows.device), arity, sum(got))

    def all_gather_rows(self, rows: torch.Tensor) -> torch.Tensor:
        """Concatenation (rank order) of every rank's rows."""
        arity, n = rows.shape
        cdev = self._dev()
        sizes = [torch.zeros(1, dtype=torch.int64, device=cdev) for _ in range(self.world)]
        self.td.all_gather(sizes, torch.tensor([n], dtype=torch.int64, device=cdev), group=self.group)
        sizes = torch.cat(sizes).tolist()  # one host read
        top = max(sizes) if sizes else 0
        mine = torch.zeros((top, arity), dtype=torch.int32, device=cdev)
        if n:
            mine[:n] = rows.view(torch.int32).t().to(cdev)
        parts = [torch.empty((top, arity), dtype=torch.int32, device=cdev) for _ in range(self.world)]
        self.td.all_gather(parts, mine, group=self.group)
        self.sent_bytes += 4 * arity * n * (self.world - 1)
        self.exchanges += 1
        got = torch.cat([p[:s] for p, s in zip(parts, sizes)]) if sizes else mine[:0]
        return got.to(rows.device).t().contiguous().view(torch.uint32)
