"""Multi-router operation: one process per GPU (router), torch.distributed for
the plumbing (reference run_detection's merge branch,
pipeline.cpp:76-85, and merge_rseas, snapshot.cpp:117-142).

Union-min (the reference default) is idempotent and commutes with
advance_slot, so every router can keep the *merged* grid: in lockstep the
merged grid changes per slot exactly by "stamp = now on every recorder any
router touched".  So routers exchange only what they touched in the slot and
fold the peers' touches into their own grid with the same kernels a single
router uses.  Three exchange formats give the same grid:

  PUSH    the slot's distinct (cip, oip) pairs, stored into the peers'
          symmetric-memory inboxes by the scan kernel itself (P2P over NVLink),
          so the exchange overlaps the scan;
  PAIRS   the same lists, all-gathered after the scan;
  BITMAP  the slot's touched bitmap (1 bit per recorder), OR-all-reduced.
  SHARD   each router owns 1/N of the cells and stamps only those; new pairs
          reach the owners of their cells over NVLink, relayed through a
          pair owner that dedups the routers' union (ShardExchange); hot bits
          are OR-merged and each survivor's in-window bucket masks AND-merged
          at reconstruction.  Per-router stamping then scales with 1/N of the
          routers' union of pairs.

SHARD, the default at N > 1, keeps the per-router counts on the device
(relay and receive kernels read them there); PUSH and PAIRS read them on the
host once per slot to size their receive scans.

merge_stamps_max is the literal all-reduce(max) of the full stamp grid, kept as
the baseline.  Every variant equals merge_rseas(node grids, kUnionMin) of the
reference bit for bit (tests/test_dist_gloo.py on CPU, tests/test_gpu_parity.py
on the device).
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def _bitwise_allreduce_nccl_(t: torch.Tensor, op: str, group=None) -> torch.Tensor:
    """Reduce-scatter by all_to_all + a local OR/AND of the received chunks,
    then all-gather: the 2(N-1)/N per-rank volume of a ring all-reduce.  The
    collective path for CPU tensors (gloo: the multi-process CPU tests)."""
    world = dist.get_world_size(group)
    flat = t.view(-1)
    n = flat.numel()
    per = (n + world - 1) // world
    padded = flat
    if per * world != n:
        padded = torch.full((per * world,), 0 if op == "or" else -1, dtype=flat.dtype, device=flat.device)
        padded[:n].copy_(flat)
    recv = torch.empty_like(padded)
    dist.all_to_all_single(recv, padded, group=group)
    chunks = recv.view(world, per)
    mine = chunks[0].clone()
    for i in range(1, world):
        (mine.bitwise_or_ if op == "or" else mine.bitwise_and_)(chunks[i])
    out = torch.empty_like(padded)
    dist.all_gather_into_tensor(out, mine, group=group)
    flat.copy_(out[:n])
    return t


class _PeerStage:
    """A symmetric-memory staging buffer per (group, device), grown on
    demand, for bitwise all-reduces by sspd_reduce_words over NVLink."""

    _cache: dict = {}

    @classmethod
    def get(cls, group, words: int, device: int):
        import torch.distributed._symmetric_memory as symm_mem

        name = group.group_name if group is not None else dist.group.WORLD.group_name
        key = (name, device)
        have = cls._cache.get(key)
        if have is not None and have[0].numel() >= words:
            return have
        buf = symm_mem.empty(max(words, 1 << 20), dtype=torch.int32, device=torch.device(f"cuda:{device}"))
        have = (buf, symm_mem.rendezvous(buf, name))
        cls._cache[key] = have
        return have


def _bitwise_allreduce_peer_(t: torch.Tensor, op: str, group=None) -> torch.Tensor:
    """In place, for a CUDA int32 tensor: every rank stages its words in a
    symmetric buffer; rank r reduces slice r from all peers' buffers with ONE
    sspd_reduce_words kernel reading over NVLink (reduce-scatter), then reads
    every other slice from its owner (all-gather).  Same 2(N-1)/N volume per
    rank as a ring all-reduce; device barriers order the phases, no host
    round trip."""
    from .grid import reduce_words

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    flat = t.view(-1)
    n = flat.numel()
    dev = flat.device.index
    buf, h = _PeerStage.get(group, n, dev)
    stream = torch.cuda.current_stream(flat.device).cuda_stream
    per = ((n + world - 1) // world + 3) // 4 * 4  # 16 B aligned slices
    lo = [min(n, p * per) for p in range(world)]
    cnt = [min(n, lo[p] + per) - lo[p] for p in range(world)]
    buf[:n].copy_(flat)
    h.barrier(channel=0)  # every rank's words staged
    if cnt[rank]:
        reduce_words(dev, [b + 4 * lo[rank] for b in h.buffer_ptrs], cnt[rank], op,
                     buf.data_ptr() + 4 * lo[rank], stream)
    h.barrier(channel=1)  # every slice reduced in its owner's buffer
    for p in range(world):
        if p != rank and cnt[p]:
            reduce_words(dev, [h.buffer_ptrs[p] + 4 * lo[p]], cnt[p], op, buf.data_ptr() + 4 * lo[p], stream)
    flat.copy_(buf[:n])
    h.barrier(channel=2)  # no peer still reads this buffer when it is next staged
    return t


def or_allreduce_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place bitwise-OR all-reduce of an int32 tensor (NCCL has no OR op):
    over peer memory for CUDA tensors, by collectives for CPU ones."""
    if dist.get_world_size(group) == 1:
        return t
    if t.is_cuda:
        return _bitwise_allreduce_peer_(t, "or", group)
    return _bitwise_allreduce_nccl_(t, "or", group)


def and_allreduce_(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place bitwise-AND all-reduce of an int32 tensor."""
    if dist.get_world_size(group) == 1:
        return t
    if t.is_cuda:
        return _bitwise_allreduce_peer_(t, "and", group)
    return _bitwise_allreduce_nccl_(t, "and", group)


class _CudaArray:
    """__cuda_array_interface__ view of raw device memory owned by the grid."""

    def __init__(self, ptr: int, n: int, typestr: str = "<i4"):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3, "strides": None}


def device_view(ptr: int, n_words: int, device: int) -> torch.Tensor:
    with torch.cuda.device(device):
        return torch.as_tensor(_CudaArray(ptr, n_words), device=f"cuda:{device}")


BITMAP = 1
PAIRS = 2
PUSH = 3
SHARD = 4


def prepare(grid, exchange: int = PAIRS, region_cap: int = 0, group=None):
    """Choose what routers exchange each slot: the slot's distinct (cip, oip)
    pairs (PAIRS, default: ~10% of a Zipf slot's packets, 8 B each), the
    same pairs pushed over NVLink during the scan (PUSH, needs region_cap =
    the most pairs a router scans per slot) or the touched bitmap (BITMAP:
    1 bit per recorder, fixed size)."""
    if exchange == PUSH:
        PushExchange(grid, region_cap, group)
        return
    if exchange == SHARD:
        ShardExchange(grid, region_cap, group)
        return
    grid.set_exchange(exchange)
    grid._exchange = exchange


def merge(grid, group=None):
    ex = getattr(grid, "_exchange", BITMAP)
    if ex == SHARD:
        grid._shard.merge(grid)
    elif ex == PUSH:
        grid._push.merge(grid)
    elif ex == PAIRS:
        merge_pairs(grid, group)
    else:
        merge_touched(grid, group)


class PushExchange:
    """Fused scan + exchange over NVLink (exchange PUSH).

    Every router owns two inboxes in torch symmetric memory (one per slot
    parity), each `world` regions of `region_cap` pairs.  While scanning, the
    dedup kernel stores each pair new to this router into region `rank` of
    every peer's current inbox (P2P stores, include/sspd_cuda.h
    sspd_set_push), so the exchange overlaps the scan.  After the scan an
    all-gather of the per-router counts is the barrier; each router then scans
    the other regions of its own inbox.  Parity double-buffering is safe: a
    router pushes slot s+2 into an inbox only after the all-gather of slot s+1,
    which the receiver joins only after it finished applying slot s.  A
    router whose slot overflows region_cap makes every router fall back to
    the all-gathered lists for that slot (the counts say so consistently).
    """

    def __init__(self, grid, region_cap: int, group=None):
        import torch.distributed._symmetric_memory as symm_mem

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.cap = int(region_cap)
        self.group = group
        dev = torch.device(f"cuda:{grid.device}")
        name = group.group_name if group is not None else dist.group.WORLD.group_name
        self.inbox, self.handles = [], []
        for _ in range(2):
            buf = symm_mem.empty(self.world * self.cap * 2, dtype=torch.int32, device=dev)
            self.inbox.append(buf)
            self.handles.append(symm_mem.rendezvous(buf, name))
        self.parity = 0
        grid.set_exchange(PAIRS)
        grid._exchange = PUSH
        grid._push = self
        self._arm(grid)

    def _arm(self, grid):
        grid.set_push(self.handles[self.parity].buffer_ptrs_dev, self.world, self.rank, self.cap)

    def merge(self, grid):
        ptr, n = grid.new_pairs_ptr()
        dev = torch.device(f"cuda:{grid.device}")
        counts = torch.tensor([n], dtype=torch.int64, device=dev)
        allc = torch.empty(self.world, dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(allc, counts, group=self.group)   # also the barrier
        sizes = [int(c) for c in allc.tolist()]
        torch.cuda.synchronize(grid.device)
        box = self.inbox[self.parity].view(self.world, self.cap, 2)
        grid.set_exchange(0)
        try:
            if max(sizes) > self.cap:
                # someone overflowed its region: everyone uses the lists
                local = (device_view(ptr, 2 * n, grid.device).view(n, 2) if n
                         else torch.zeros((0, 2), dtype=torch.int32, device=dev))
                for part in exchange_pairs(local, self.group):
                    grid.scan_device(part.data_ptr(), int(part.shape[0]))
            else:
                for src in range(self.world):
                    if src != self.rank and sizes[src]:
                        grid.scan_device(box[src].data_ptr(), sizes[src])
        finally:
            grid.set_exchange(PAIRS)
        self.parity ^= 1
        self._arm(grid)


def reconstruct(grid, k: int, theta: float, group=None):
    """reconstruct_leveled on the merged grid, for every exchange: sharded
    routers merge their hot bits and survivor masks (ShardExchange); the
    others hold the merged grid already."""
    if getattr(grid, "_exchange", None) == SHARD:
        return grid._shard.reconstruct(grid, k, theta)
    return grid.reconstruct_leveled(k, theta)


class ShardExchange:
    """Sharded union-min (exchange SHARD; include/sspd_cuda.h "sharded
    routers").

    Router `rank` owns the cells c with c * world // (r * 2^q) == rank and
    keeps exact stamps only there.  relay=True (the default) routes pairs in
    two hops through symmetric-memory inboxes (P2P stores over NVLink, double
    buffered by slot parity as in PushExchange):

      scan    each pair new to a router goes to its pair owner
              (a hash of the pair mod world; inboxes A);
      merge   an all-gather of the hop-1 counts is the barrier; every pair
              owner dedups what it received (the routers' union, for its
              share), stamps its own cells and pushes each pair once to the
              other cell owners (inboxes B); a second all-gather; every
              router stamps what was relayed to it.

    relay=False pushes straight from the scan to every other cell owner (one
    hop; a pair several routers saw then reaches its owners several times).
    Measured on one GPU with all routers' work in lockstep
    (profiles/r01_shard_sim.md): a router's slot at N=8 is 4.0 ms relayed,
    6.4 ms one-hop, 11.7 ms with the replicated PAIRS exchange.

    reconstruct(): OR-all-reduce of the routers' hot bits (r * 2^q bits), the
    same joins on every router, AND-all-reduce of the per-survivor bucket
    masks (n_surv * eta bits), popcount -- the reports equal reconstruct on the
    union-min merged grid.  region_cap must cover the pairs a router scans per
    slot plus list padding (kernels.cuh list_pad); a count past it raises.

    No host round trip inside merge(): the per-router counts are all-gathered
    on the device and the relay/receive kernels read them from device memory
    (sspd_shard_*_regions_dev); stream order (the grid's stream joined to
    torch's around each collective) is the only synchronisation.  The hot-bit
    OR and the mask AND run as ONE kernel per router over the peers'
    symmetric-memory copies (sspd_reduce_words over NVLink) after a device
    barrier of the symmetric-memory handle; buffers alternate by slot parity.
    """

    MASK_WORDS = 1 << 22  # symmetric mask buffer (16 MiB); more survivors fall back to NCCL

    def __init__(self, grid, region_cap: int, group=None, relay: bool = True):
        import torch.distributed._symmetric_memory as symm_mem

        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.cap = int(region_cap)
        self.group = group
        self.relay = relay
        dev = torch.device(f"cuda:{grid.device}")
        name = group.group_name if group is not None else dist.group.WORLD.group_name
        self.inbox, self.handles = [], []  # [parity][hop]
        for _ in range(2):
            bufs, hs = [], []
            for _ in range(2 if relay else 1):
                buf = symm_mem.empty(self.world * self.cap * 2, dtype=torch.int32, device=dev)
                bufs.append(buf)
                hs.append(symm_mem.rendezvous(buf, name))
            self.inbox.append(bufs)
            self.handles.append(hs)
        self.parity = 0
        # per parity: symmetric copies of the hot bits and of the survivor masks
        hot_words = grid.r * (((1 << grid.q) + 31) // 32)
        self.hot_sym, self.mask_sym = [], []
        for _ in range(2):
            hb = symm_mem.empty(hot_words, dtype=torch.int32, device=dev)
            mb = symm_mem.empty(self.MASK_WORDS, dtype=torch.int32, device=dev)
            self.hot_sym.append((hb, symm_mem.rendezvous(hb, name)))
            self.mask_sym.append((mb, symm_mem.rendezvous(mb, name)))
        self._keep = []  # count tensors the queued kernels still read
        grid._exchange = SHARD
        grid._shard = self
        self._arm(grid)

    def _arm(self, grid):
        hs = self.handles[self.parity]
        if self.relay:
            grid.set_shard_relay(hs[0].buffer_ptrs_dev, hs[1].buffer_ptrs_dev, self.world, self.rank, self.cap)
        else:
            grid.set_shard(hs[0].buffer_ptrs_dev, self.world, self.rank, self.cap)

    def _streams(self, grid):
        dev = torch.device(f"cuda:{grid.device}")
        return torch.cuda.current_stream(dev), torch.cuda.ExternalStream(grid.stream_handle(), device=dev)

    def _counts(self, grid, hop: int) -> torch.Tensor:
        """sent[src][dst] of hop 0 or 1, all-gathered on the device (also the
        barrier: every router's pushes precede its contribution in stream
        order, and the kernels fence them system-wide).  Row-major
        [src * world + dst]; no host copy."""
        cur, gs = self._streams(grid)
        cur.wait_stream(gs)  # this router's scan/relay kernels, then the collective
        mine = device_view(grid.shard_sent_ptr(), 128, grid.device).view(torch.int64)
        mine = mine[32 * hop: 32 * hop + self.world].clone()
        allsent = torch.empty(self.world * self.world, dtype=torch.int64, device=mine.device)
        dist.all_gather_into_tensor(allsent, mine, group=self.group)
        gs.wait_stream(cur)  # the next kernels read the gathered counts
        self._keep.append(allsent)
        return allsent

    def merge(self, grid):
        self._keep = []
        bufs = self.inbox[self.parity]
        col = lambda t: t.data_ptr() + 8 * self.rank  # noqa: E731 -- counts [src][rank], stride world
        if self.relay:
            sent = self._counts(grid, 0)
            # the routers' pairs routed here (this router's own included), all regions in one launch
            grid.shard_relay_regions_dev(bufs[0].data_ptr(), self.cap, col(sent), self.world, self.world)
            sent = self._counts(grid, 1)
            box = bufs[1]
        else:
            sent = self._counts(grid, 0)
            box = bufs[0]
        # every other router's region of this router's inbox, one launch
        grid.shard_receive_regions_dev(box.data_ptr(), self.cap, col(sent), self.world, self.world, self.rank)
        self.parity ^= 1
        self._arm(grid)

    def _reduce_peers(self, grid, src_ptr: int, words: int, sym, op: str):
        """In place: the words at src_ptr become the OR/AND over all routers',
        read from the peers' symmetric copies by one kernel."""
        buf, h = sym
        cur, gs = self._streams(grid)
        cur.wait_stream(gs)
        buf[:words].copy_(device_view(src_ptr, words, grid.device))
        h.barrier(channel=self.parity)  # every router's copy is in place
        from .grid import reduce_words
        reduce_words(grid.device, list(h.buffer_ptrs), words, op, src_ptr, cur.cuda_stream)
        gs.wait_stream(cur)

    def reconstruct(self, grid, k: int, theta: float):
        p = self.parity
        ptr, n = grid.shard_hot(k, theta)
        if grid.shard_overflow():
            raise RuntimeError(f"shard exchange: pairs for one owner exceed region_cap {self.cap}")
        self._reduce_peers(grid, ptr, n, self.hot_sym[p], "or")
        ns, mptr, words = grid.shard_select(k, theta)
        if ns:
            if words <= self.MASK_WORDS:
                self._reduce_peers(grid, mptr, words, self.mask_sym[p], "and")
            else:
                and_allreduce_(device_view(mptr, words, grid.device), self.group)
                torch.cuda.synchronize(grid.device)
        return grid.shard_finish(theta)


def exchange_pairs(local: torch.Tensor, group=None) -> list[torch.Tensor]:
    """All-gather variable-length (n, 2) int32 pair lists; returns the other
    ranks' lists (views into one receive buffer), in rank order."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = local.shape[0]
    counts = torch.tensor([n], dtype=torch.int64, device=local.device)
    all_counts = torch.empty(world, dtype=torch.int64, device=local.device)
    dist.all_gather_into_tensor(all_counts, counts, group=group)
    sizes = [int(c) for c in all_counts.tolist()]
    width = max(sizes) if sizes else 0
    if width == 0:
        return []
    mine = torch.zeros((width, 2), dtype=torch.int32, device=local.device)
    if n:
        mine[:n].copy_(local)
    everyone = torch.empty((world * width, 2), dtype=torch.int32, device=local.device)
    dist.all_gather_into_tensor(everyone, mine, group=group)
    return [everyone[r * width: r * width + sizes[r]] for r in range(world) if r != rank and sizes[r]]


def merge_pairs(grid, group=None):
    """Union-min merge by pair lists: all-gather every router's distinct
    pairs of the slot and scan the other routers' lists locally.  The union
    of the touches equals the union-min merge of the node grids; the grid's
    pair set skips pairs this router already saw."""
    if dist.get_world_size(group) == 1:
        return
    ptr, n = grid.new_pairs_ptr()
    dev = torch.device(f"cuda:{grid.device}")
    local = (device_view(ptr, 2 * n, grid.device).view(n, 2) if n
             else torch.zeros((0, 2), dtype=torch.int32, device=dev))
    remote = exchange_pairs(local, group)
    torch.cuda.synchronize(grid.device)
    grid.set_exchange(0)  # remote pairs are not re-exported
    try:
        for part in remote:
            grid.scan_device(part.data_ptr(), int(part.shape[0]))
    finally:
        grid.set_exchange(PAIRS)


def merge_touched(grid, group=None):
    """Union-min merge of this slot's touches across routers (in place)."""
    ptr, n = grid.touched_ptr()
    bits = device_view(ptr, n, grid.device)
    or_allreduce_(bits, group)
    torch.cuda.synchronize(grid.device)  # the grid's stream may differ from torch's
    grid.commit()


def merge_stamps_max(grid, group=None):
    """The literal north-star merge: all-reduce(max) of the full stamp grid.
    Correct but moves 32x the bytes of merge_touched; kept for comparison."""
    ptr, n = grid.stamps_ptr()
    st = device_view(ptr, n, grid.device)
    dist.all_reduce(st, op=dist.ReduceOp.MAX, group=group)
