"""Head-parallel MPIC-k prefill of one long request over P GPUs.

Rank r of P owns heads [r*H/P, (r+1)*H/P). Per layer:

  1. engine.attn(l)      QKV projection of its heads (+RoPE, KV scatter into its head slice of
                         the request cache), attention over its heads, and its share of
                         attn . Wo^T: an fp32 partial sum of all h outputs for the m rows;
  2. reduce-scatter      partials summed over the ranks; rank r receives rows [r*mr, (r+1)*mr)
                         (m padded to m_pad = P*mr with zero rows);
  3. engine.ffn(l, ...)  residual add of those rows, then W1+GELU and W2+residual on its
                         m/P rows only (full FFN weights, 1/P of the FFN FLOPs);
  4. all-gather          the bf16 rows (the next layer's QKV input) back to every rank.

Steps 2+4 move the bytes of one all-reduce per layer (the north star's "one NCCL all-reduce
per layer") without replicating the FFN. The rank holding row m-1 computes the logits.

Two drivers:
  * `HeadParallelRank.request(..., comm=NcclComm)` — the production path: the whole request
    runs inside the library (mpic_hp_request): the layer loop, the NCCL reduce-scatter /
    all-gather and the logits broadcast are issued by C++ on the caller's stream, and the
    loop is captured as one CUDA graph for same-shape requests. NcclComm is a communicator
    the library creates (mpic_nccl_comm_create) from an id rank 0 distributes.
  * `prefill_layers(engine, comm)` — the same decomposition step by step from Python with
    the collectives of `TorchComm` (torch.distributed: NCCL between GPUs, gloo on CPU or
    between processes sharing a GPU); `prefill_local` runs P virtual ranks on one GPU in
    lockstep. These exercise the row split / padding / owner logic on any backend.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import PolicyDesc, check, lib


def row_split(m: int, world: int):
    """(mr, m_pad): rows per rank and the padded row count, m_pad = world * mr >= m."""
    mr = -(-m // world)
    return mr, mr * world


class TorchComm:
    """Collectives over torch.distributed (NCCL between GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist, self.group = dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

        self.nccl = dist.get_backend(group) == "nccl"

    def reduce_scatter(self, partial, out):
        """out (mr x h) = rows [rank*mr, (rank+1)*mr) of the sum over ranks of partial."""
        if self.nccl:
            self.dist.reduce_scatter_tensor(out, partial, op=self.dist.ReduceOp.SUM, group=self.group)
        else:  # gloo has no reduce-scatter: all-reduce a copy and keep this rank's rows
            tot = partial.clone()
            self.dist.all_reduce(tot, op=self.dist.ReduceOp.SUM, group=self.group)
            mr = out.shape[0]
            out.copy_(tot[self.rank * mr:(self.rank + 1) * mr])

    def all_gather_rows(self, full, mr):
        """All-gather of rank r's rows [r*mr, (r+1)*mr) of `full` into every rank's `full`."""
        mine = full[self.rank * mr:(self.rank + 1) * mr].clone()
        if self.nccl:
            self.dist.all_gather_into_tensor(full, mine, group=self.group)
        else:  # gloo has no 16-bit integer type: move bf16 bit patterns as int32 pairs
            import torch
            wide = mine.element_size() == 2 and mine.shape[-1] % 2 == 0
            mine_w = mine.view(torch.int32) if wide else mine
            parts = [torch.empty_like(mine_w) for _ in range(self.world)]
            self.dist.all_gather(parts, mine_w, group=self.group)
            for r in range(self.world):
                full[r * mr:(r + 1) * mr].copy_(parts[r].view(mine.dtype) if wide else parts[r])


class SoloComm:
    """world_size 1: the collectives are identities."""
    rank, world = 0, 1

    def reduce_scatter(self, partial, out):
        out.copy_(partial[:out.shape[0]])

    def all_gather_rows(self, full, mr):
        pass


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (mpic_nccl_unique_id), as bytes."""
    buf = (C.c_uint8 * 128)()
    check(lib().mpic_nccl_unique_id(buf))
    return bytes(buf)


class NcclComm:
    """An NCCL communicator created by the library (mpic_nccl_comm_create) for
    mpic_hp_request. Rank 0's id reaches the other ranks through torch.distributed
    (broadcast_object_list on `group`, any backend) unless `uid` is given."""

    def __init__(self, rank: int, world: int, device: int = 0, uid: bytes | None = None, group=None):
        if uid is None:
            if world == 1:
                uid = nccl_unique_id()
            else:
                import torch.distributed as dist
                box = [nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(box, src=0, group=group)
                uid = box[0]
        self.rank, self.world = rank, world
        h = C.c_void_p()
        check(lib().mpic_nccl_comm_create((C.c_uint8 * 128).from_buffer_copy(uid), world, rank, device, C.byref(h)))
        self.handle = h.value

    def close(self):
        if getattr(self, "handle", None):
            lib().mpic_nccl_comm_destroy(self.handle)
            self.handle = None

    __del__ = close


class _DevArray:
    """__cuda_array_interface__ view of a raw device pointer (torch.as_tensor aliases it)."""

    def __init__(self, ptr, shape, typestr):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3, "strides": None}


def device_tensor(ptr, shape, dtype):
    import torch
    typestr = {torch.float32: "<f4", torch.int16: "<i2"}[dtype]
    return torch.as_tensor(_DevArray(ptr, shape, typestr), device="cuda")


class HeadParallelRank:
    """One rank's share of a head-parallel request on the B200 library."""

    def __init__(self, cfg, rank: int, world: int, device: int = 0, max_rows: int = 2048,
                 max_ctx: int = 0):
        from . import BF16, Workspace
        if cfg.n_heads % world:
            raise ValueError("heads must divide evenly over the ranks")
        self.cfg, self.rank, self.world, self.device = cfg, rank, world, device
        self.hl = cfg.n_heads // world
        self.head0 = rank * self.hl
        h = C.c_void_p()
        check(lib().mpic_model_create_heads(C.byref(cfg), device, BF16, self.head0, self.hl,
                                            C.byref(h)))

        class _M:  # minimal stand-in so Workspace/KV helpers accept the slice model
            pass
        self.model = _M()
        self.model.handle, self.model.cfg, self.model.dtype = h.value, cfg, BF16
        self.ws = Workspace(self.model, max_rows, max_ctx)
        self.ws_rows = -(-max_rows // 128) * 128  # the workspace's padded row capacity

    def close(self):
        if getattr(self, "ws", None):
            self.ws.close()
            self.ws = None
        if getattr(self, "model", None) and self.model.handle:
            lib().mpic_model_destroy(self.model.handle)
            self.model.handle = None

    __del__ = close

    def linked_cache(self, n: int):
        from . import BF16, KV
        return KV(self.cfg.n_layers, n, self.hl, self.cfg.head_dim, BF16, self.device)

    # ---- engine interface used by prefill_layers() --------------------------------------
    def prepare(self, prompt, chunks, linked, policy, k, stream, reposition=0, position_bases=None):
        import torch
        n_img = len(chunks)
        arr = (C.c_void_p * max(n_img, 1))(*[c.handle for c in chunks])
        pb = np.ascontiguousarray(position_bases if position_bases is not None else np.zeros(n_img),
                                  np.uint32)
        sel = np.zeros(prompt.n, np.uint32)
        m = C.c_uint32()
        pol = PolicyDesc(policy, k, 0)
        self._stream = stream
        check(lib().mpic_hp_prepare(self.model.handle, self.ws.handle, C.byref(prompt.desc()),
                                    C.byref(pol), arr, reposition, pb.ctypes.data, linked.handle,
                                    sel.ctypes.data, C.byref(m), stream))
        self.m = m.value
        self.linked = linked
        self.mr, self.m_pad = row_split(self.m, self.world)
        if self.m_pad > self.ws_rows:  # the all-gather writes m_pad rows of the workspace's xb
            raise ValueError(f"{self.world} x ceil(m/{self.world}) = {self.m_pad} rows exceed the workspace "
                             f"({self.ws_rows}): create the rank with max_rows >= m + world")
        h = self.cfg.hidden_dim
        self.partial = torch.zeros(self.m_pad, h, dtype=torch.float32, device=f"cuda:{self.device}")
        self.reduced = torch.zeros(self.mr, h, dtype=torch.float32, device=f"cuda:{self.device}")
        p = C.c_void_p()
        check(lib().mpic_workspace_device_ptr(self.ws.handle, 1, C.byref(p)))
        self.xb_all = device_tensor(p.value, (self.m_pad, h), torch.int16)  # bf16 bits
        return sel[:self.m].copy()

    def request(self, prompt, chunks, linked, k: int = 32, stream=None, comm: NcclComm | None = None,
                policy: int = 0, reposition: int = 0, position_bases=None):
        """The whole head-parallel request in the library (mpic_hp_request): every rank gets
        the logits. comm=None runs P = 1 (this rank must own every head)."""
        n_img = len(chunks)
        arr = (C.c_void_p * max(n_img, 1))(*[c.handle for c in chunks])
        pb = np.ascontiguousarray(position_bases if position_bases is not None else np.zeros(n_img),
                                  np.uint32)
        sel = np.zeros(prompt.n, np.uint32)
        logits = np.zeros(self.cfg.vocab_size, np.float32)
        m = C.c_uint32()
        pol = PolicyDesc(policy, k, 0)
        check(lib().mpic_hp_request(self.model.handle, self.ws.handle, comm.handle if comm else None,
                                    C.byref(prompt.desc()), C.byref(pol), arr, reposition, pb.ctypes.data,
                                    linked.handle, logits.ctypes.data, sel.ctypes.data, C.byref(m), stream))
        self.m = m.value
        return logits, sel[:self.m].copy()

    def attn(self, layer):
        check(lib().mpic_hp_layer_attn(self.model.handle, self.ws.handle, layer, self.linked.handle,
                                       self.partial.data_ptr(), self._stream))

    def ffn(self, layer, reduced, row0, rows):
        check(lib().mpic_hp_layer_ffn(self.model.handle, self.ws.handle, layer, reduced.data_ptr(),
                                      row0, rows, self._stream))

    def logits(self, row):
        out = np.zeros(self.cfg.vocab_size, np.float32)
        check(lib().mpic_hp_logits(self.model.handle, self.ws.handle, row, out.ctypes.data,
                                   self._stream))
        return out


def prefill_layers(engine, comm, n_layers: int):
    """Steps 1-4 of the module docstring for every layer on one rank; returns the logits on
    the rank holding row m-1, else None."""
    mr = engine.mr
    for layer in range(n_layers):
        engine.attn(layer)
        comm.reduce_scatter(engine.partial, engine.reduced)
        engine.ffn(layer, engine.reduced, comm.rank * mr, mr)
        comm.all_gather_rows(engine.xb_all, mr)
    last = engine.m - 1
    return engine.logits(last) if last // mr == comm.rank else None


def prefill_local(engines, n_layers: int):
    """Run a head-parallel request on P virtual ranks sharing one GPU, layer by layer in
    lockstep (the parity test of the decomposition on a single device)."""
    import torch
    world = len(engines)
    mr = engines[0].mr
    for layer in range(n_layers):
        for e in engines:
            e.attn(layer)
        total = sum(e.partial for e in engines)  # reduce ...
        for r, e in enumerate(engines):          # ... scatter
            e.reduced.copy_(total[r * mr:(r + 1) * mr])
            e.ffn(layer, e.reduced, r * mr, mr)
        gathered = torch.cat([e.xb_all[r * mr:(r + 1) * mr] for r, e in enumerate(engines)])
        for e in engines:                         # all-gather
            e.xb_all.copy_(gathered)
    torch.cuda.synchronize()
    last = engines[0].m - 1
    return engines[last // mr].logits(last)
