"""Row-sharded QTIP linear layer across ranks (BASELINE config C4).

Each rank owns a contiguous range of output rows (a multiple of 128 = one cell row block),
computes scale * W~[rows] x~ with qtip_matvec (RHT-in on the replicated x, RHT-out off),
the shards are exchanged with one all-gather over NCCL (NVLink 5 / NVSwitch), and every
rank applies the inverse output RHT y = S_m H_m^T y~ / sqrt(m) (it mixes all rows, so it
cannot be split).  With kernels 1-6 per-row arithmetic is unchanged by sharding (the gathered
y~ equals the single-GPU y~ bit for bit); the stream-K kernel (7) partitions each shard's own
cells, so there the agreement is to fp32 rounding (include/qtip.h).
"""
import numpy as np

CELL_ROWS = 128


def shard_rows(m, world):
    """Contiguous row ranges, multiples of 128 except the last; sizes differ by <= 128."""
    nrb = (m + CELL_ROWS - 1) // CELL_ROWS
    out = []
    start_rb = 0
    for r in range(world):
        cnt = nrb // world + (1 if r < nrb % world else 0)
        r0 = min(start_rb * CELL_ROWS, m)
        r1 = min((start_rb + cnt) * CELL_ROWS, m)
        out.append((r0, r1))
        start_rb += cnt
    return out


def padded_shard_rows(m, world):
    """Equal per-rank slot size for all_gather_into_tensor."""
    return max(r1 - r0 for r0, r1 in shard_rows(m, world))


def gather_order(slots, m, world):
    """Indices that turn the gathered [world, slot] buffer into the m rows (drops padding)."""
    idx = []
    for r, (r0, r1) in enumerate(shard_rows(m, world)):
        idx.extend(range(r * slots, r * slots + (r1 - r0)))
    return np.array(idx, dtype=np.int64)


def gather_rows(send, recv, world, m, group=None, out=None):
    """The exchange step: every rank's padded y~ slice send [B, slot] -> y~ [B, m] in row order on
    every rank (one all_gather_into_tensor; NCCL on GPUs, gloo in the CPU tests).  recv is the
    [world, B, slot] staging buffer; out (optional) receives the reordered rows."""
    import torch
    import torch.distributed as dist
    B, slot = send.shape
    dist.all_gather_into_tensor(recv.view(-1), send.reshape(-1), group=group)
    if B == 1 and slot * world == m:
        return recv.view(1, m)                                           # already in row order
    idx = torch.from_numpy(gather_order(slot, m, world)).to(send.device)
    rows = recv.permute(1, 0, 2).reshape(B, -1).index_select(1, idx)    # drop padding, reorder
    if out is None:
        return rows
    out.copy_(rows)
    return out


class ShardedQTIPLinear:
    """One rank's part of a row-sharded layer.  `group` is a torch.distributed process group."""

    def __init__(self, m, n, rank, world, code="3inst", k=2, device="cuda", group=None):
        import torch
        from .layer import QTIPLinear
        self.m, self.n, self.rank, self.world, self.group = m, n, rank, world, group
        self.rows = shard_rows(m, world)[rank]
        self.slot = padded_shard_rows(m, world)
        self.local = QTIPLinear(self.rows[1] - self.rows[0], n, code=code, k=k, device=device)
        self.sign_m = torch.zeros((m + 7) // 8, dtype=torch.uint8, device=device)
        self.scale = 1.0
        self._bufs = {}
        self.device = device

    def load_tiles(self, tiles_full_or_shard, sign_m, sign_n, scale=1.0, lut=None, is_shard=False):
        import torch
        r0, r1 = self.rows
        tiles = tiles_full_or_shard if is_shard else tiles_full_or_shard[r0 // 16:r1 // 16]
        self.local.load_tiles(tiles, np.zeros((r1 - r0 + 7) // 8, np.uint8), sign_n, scale=scale, lut=lut)
        self.sign_m.copy_(torch.from_numpy(np.ascontiguousarray(sign_m, dtype=np.uint8)))
        self.scale = scale
        return self

    def _buffers(self, B):
        import torch
        if B not in self._bufs:
            send = torch.zeros((B, self.slot), dtype=torch.float32, device=self.device)
            recv = torch.empty((self.world, B, self.slot), dtype=torch.float32, device=self.device)
            yt = torch.empty((B, self.m), dtype=torch.float32, device=self.device)
            y = torch.empty((B, self.m), dtype=torch.float32, device=self.device)
            idx = torch.from_numpy(gather_order(self.slot, self.m, self.world)).to(self.device)
            tmp = torch.empty((B, self.rows[1] - self.rows[0]), dtype=torch.float32, device=self.device)
            self._bufs[B] = (send, recv, yt, y, idx, tmp)
        return self._bufs[B]

    def forward(self, x):
        from . import qtip
        B = x.shape[0]
        send, recv, yt, y, idx, tmp = self._buffers(B)
        rows = self.rows[1] - self.rows[0]
        if rows == self.slot:
            self.local.forward(x, out=send, flags=qtip.QTIP_RHT_IN)      # scale * W~[rows] x~
        else:
            self.local.forward(x, out=tmp, flags=qtip.QTIP_RHT_IN)
            send[:, :rows].copy_(tmp)
        src = gather_rows(send, recv, self.world, self.m, group=self.group, out=yt)
        qtip.qtip_rht(self.m, B, self.sign_m, src, y, inverse=True)          # S_m H_m^T y~ / sqrt(m)
        return y

    __call__ = forward
