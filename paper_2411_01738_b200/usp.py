"""Thin ctypes binding of libxdit_usp.so (include/xdit_usp.h).

Argument marshalling only: torch tensors -> device pointers, the current CUDA stream -> handle,
status codes -> exceptions.  Every step of the hot path runs in the library's CUDA kernels and
NCCL; there is no Python or CPU fallback -- if the extension is missing this module raises.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("XDIT_LIB") or os.path.join(HERE, "libxdit_usp.so")  # XDIT_LIB: A/B builds

XDIT_STATUS = {0: "OK", 1: "INVALID_ARG", 2: "UNSUPPORTED", 3: "DIVISIBILITY", 4: "COMM_MISMATCH",
               5: "EMPTY_SHARD", 6: "ALIGNMENT", 7: "CUDA", 8: "NCCL", 9: "WORKSPACE", 10: "NOT_CONNECTED"}
NCCL_UNIQUE_ID_BYTES = 128
PEER_BLOB_BYTES = 1024  # XDIT_PEER_BLOB_BYTES
TRANSPORTS = {"nccl": 0, "peer": 1}  # XDIT_TRANSPORT_NCCL / XDIT_TRANSPORT_PEER


class XditError(RuntimeError):
    def __init__(self, code: int, fn: str, msg: str):
        self.code = code
        self.status = XDIT_STATUS.get(code, str(code))
        super().__init__(f"{fn} -> XDIT_ERR_{self.status} ({code}): {msg}")


class RowMap(ctypes.Structure):
    """xdit_rowmap: destination of an output row block (see include/xdit_usp.h)."""
    _fields_ = [("nseg", ctypes.c_int32), ("seg_off", ctypes.c_int32 * 9),
                ("o_seg", ctypes.c_int64), ("o_b", ctypes.c_int64), ("o_s", ctypes.c_int64),
                ("o_h", ctypes.c_int64), ("l_seg", ctypes.c_int64), ("l_b", ctypes.c_int64),
                ("l_h", ctypes.c_int64), ("o_seg_off", ctypes.c_int64 * 8), ("l_seg_off", ctypes.c_int64 * 8),
                ("seg_table", ctypes.c_int32)]

    @classmethod
    def plain(cls, B: int, S: int, H: int, D: int) -> "RowMap":
        """A plain [B][S][H][D] output with lse [B][H][S]."""
        m = cls()
        m.nseg = 1
        m.seg_off[1] = S
        m.o_b, m.o_s, m.o_h = S * H * D, H * D, D
        m.l_b, m.l_h = H * S, S
        return m


class Plan(ctypes.Structure):
    """xdit_plan: per-rank geometry of one USP call."""
    _fields_ = [("nranks", ctypes.c_int32), ("rank", ctypes.c_int32), ("ulysses", ctypes.c_int32),
                ("ring", ctypes.c_int32), ("i", ctypes.c_int32), ("j", ctypes.c_int32),
                ("Hh", ctypes.c_int32), ("S_loc", ctypes.c_int32), ("Lmax", ctypes.c_int32),
                ("S_blk", ctypes.c_int32), ("ring_next", ctypes.c_int32), ("ring_prev", ctypes.c_int32),
                ("nseg", ctypes.c_int32), ("seg_off", ctypes.c_int32 * 9),
                ("ring_src", ctypes.c_int32 * 8), ("ring_rows", ctypes.c_int32 * 8),
                ("a2a_bytes_per_peer", ctypes.c_int64), ("ring_bytes", ctypes.c_int64 * 8)]


_lib = None
_vp, _i, _i64, _fp = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_void_p

_SIGS = {
    "xdit_last_error": ([], ctypes.c_char_p),
    "xdit_version": ([], _i),
    "xdit_launch_count": ([], ctypes.c_uint64),
    "xdit_usp_shard": ([_i, _i, _i, _i] + [ctypes.POINTER(_i)] * 4, _i),
    "xdit_usp_plan": ([_i] * 8 + [ctypes.POINTER(Plan)], _i),
    "xdit_nccl_unique_id": ([_vp], _i),
    "xdit_comm_init": ([_vp, _i, _i, _i, _i, ctypes.POINTER(_vp)], _i),
    "xdit_comm_create": ([_vp, _i, _i, ctypes.POINTER(_vp)], _i),
    "xdit_comm_init_peer": ([_i, _i, _i, _i, ctypes.POINTER(_vp)], _i),
    "xdit_comm_peer_export": ([_vp, _vp], _i),
    "xdit_comm_peer_connect": ([_vp, _vp], _i),
    "xdit_comm_transport": ([_vp], _i),
    "xdit_comm_mailbox_reserve": ([_vp, ctypes.c_size_t], _i),
    "xdit_p2p_mailbox": ([_vp, _i, ctypes.POINTER(_vp), ctypes.POINTER(ctypes.c_size_t)], _i),
    "xdit_p2p_put": ([_vp, _i, _vp, ctypes.c_size_t, ctypes.c_size_t, ctypes.c_uint32, _vp], _i),
    "xdit_p2p_wait": ([_vp, _i, ctypes.c_uint32, _vp], _i),
    "xdit_p2p_ack": ([_vp, _i, ctypes.c_uint32, _vp], _i),
    "xdit_p2p_wait_ack": ([_vp, _i, ctypes.c_uint32, _vp], _i),
    "xdit_comm_reserve": ([_vp, _i, _i, _i, _i, _i, _i], _i),
    "xdit_comm_info": ([_vp] + [ctypes.POINTER(_i)] * 4, _i),
    "xdit_comm_destroy": ([_vp], _i),
    "xdit_usp_attention": ([_vp] * 5 + [_i] * 7 + [_vp, _vp], _i),
    "xdit_usp_attention_f32": ([_vp] * 5 + [_i] * 7 + [_vp, _vp], _i),
    "xdit_usp_attention_kv": ([_vp] * 6 + [_i] * 7 + [_vp, _vp], _i),
    "xdit_cfg_combine": ([_vp, _vp, _vp, _i64, ctypes.c_float, _i, _vp], _i),
    "xdit_cfg_tail": ([_vp, _vp, _vp, _i64, ctypes.c_float, _i, _vp, _vp], _i),
    "xdit_kv_retain": ([_vp, _vp, _vp] + [_i] * 6 + [_i64] * 3 + [_i, _vp], _i),
    "xdit_attn_fwd": ([_vp] * 5 + [_i] * 5 + [_i64] * 6 + [ctypes.POINTER(RowMap), _i, _i, _vp, ctypes.c_size_t,
                                                            _vp], _i),
    "xdit_attn_scratch_bytes": ([_i], ctypes.c_size_t),
    "xdit_lse_merge": ([_vp] * 4 + [_i] * 4 + [_vp, _vp, ctypes.POINTER(RowMap), _i, _vp], _i),
    "xdit_uly_pack": ([_vp, _vp] + [_i] * 9 + [_vp], _i),
    "xdit_uly_unpack": ([_vp, _vp] + [_i] * 5 + [ctypes.POINTER(_i), _i, _i, _i, _vp], _i),
    "xdit_uly_unpack_out": ([_vp, _vp, _i64, _i64, _vp, _vp] + [_i] * 7 + [_vp], _i),
    "xdit_pf_block_workspace_bytes": ([_i] * 5, ctypes.c_size_t),
    "xdit_pf_block": ([_vp] * 4 + [ctypes.c_size_t] + [_i] * 7 + [_vp], _i),
    "xdit_pf_sampler": ([_vp, _vp, _i64, ctypes.c_float, _i, _vp], _i),
    "xdit_vae_conv3x3": ([_vp, _i, _i, _i, _vp, _vp, _vp, _i, _i, _vp], _i),
    "xdit_vae_conv3x3_bf16": ([_vp, _i, _i, _i, _vp, _vp, _vp, _i, _i, _vp], _i),
}


def lib():
    """Load libxdit_usp.so (built in-tree by paper_2411_01738_b200.build); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2411_01738_b200.build` "
                              "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (args, res) in _SIGS.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _lib = L
    return _lib


def _check(rc: int, fn: str):
    if rc != 0:
        raise XditError(rc, fn, lib().xdit_last_error().decode(errors="replace"))


def last_error() -> str:
    return lib().xdit_last_error().decode(errors="replace")


def version() -> int:
    return int(lib().xdit_version())


def launch_count() -> int:
    """Kernels this library has launched in this process (xdit_launch_count)."""
    return int(lib().xdit_launch_count())


def exported_symbols() -> Sequence[str]:
    return list(_SIGS)


# ------------------------------------------------------------------------------------ host logic
def shard(S_txt: int, S_img: int, nranks: int, g: int) -> Tuple[int, int, int, int]:
    """(txt_off, txt_len, img_off, img_len) of SP rank g (reading C5)."""
    v = [_i() for _ in range(4)]
    _check(lib().xdit_usp_shard(S_txt, S_img, nranks, g, *[ctypes.byref(x) for x in v]), "xdit_usp_shard")
    return tuple(int(x.value) for x in v)


def plan(B: int, H: int, S_txt: int, S_img: int, D: int, ulysses: int, ring: int, rank: int) -> Plan:
    p = Plan()
    _check(lib().xdit_usp_plan(B, H, S_txt, S_img, D, ulysses, ring, rank, ctypes.byref(p)), "xdit_usp_plan")
    return p


# ------------------------------------------------------------------------------------ torch glue
def _ptr(t) -> Optional[int]:
    """Device pointer of a tensor (or a raw integer address, passed through)."""
    if t is None or isinstance(t, int):
        return t
    return t.data_ptr()


def _stream(stream=None) -> int:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


class Comm:
    """One SP group (= one CFG group): ulysses x ring mesh, transport, workspace.

    transport="peer" (default): the library's peer-memory transport -- ranks map each other's
    receive buffers (CUDA IPC over NVLink/NVSwitch) and order their streams with device flags;
    torch.distributed (`group`, any backend) only carries the one-time handle exchange.
    transport="nccl": rank 0 of `group` creates an NCCL unique id, broadcast with torch.distributed,
    and every rank calls xdit_comm_init (the library's own NCCL communicators).
    With ulysses*ring == 1 neither is needed and no communication object is made.
    """

    def __init__(self, ulysses: int = 1, ring: int = 1, group=None, transport: str = "peer"):
        if transport not in TRANSPORTS:
            raise XditError(1, "Comm", f"transport must be one of {sorted(TRANSPORTS)}, got {transport!r}")
        self.ulysses, self.ring, self.group = ulysses, ring, group
        n = ulysses * ring
        h = _vp()
        self.transport = transport if n > 1 else "nccl"
        if n == 1:
            _check(lib().xdit_comm_init(None, 1, 0, 1, 1, ctypes.byref(h)), "xdit_comm_init")
            self.rank = 0
        else:
            import torch.distributed as dist
            rank = dist.get_rank(group)
            if dist.get_world_size(group) != n:
                raise XditError(4, "Comm", f"group size {dist.get_world_size(group)} != ulysses*ring={n}")
            if transport == "peer":
                _check(lib().xdit_comm_init_peer(n, rank, ulysses, ring, ctypes.byref(h)), "xdit_comm_init_peer")
            else:
                buf = (ctypes.c_uint8 * NCCL_UNIQUE_ID_BYTES)()
                if rank == 0:
                    _check(lib().xdit_nccl_unique_id(ctypes.cast(buf, _vp)), "xdit_nccl_unique_id")
                obj = [bytes(buf)]
                src = dist.get_global_rank(group, 0) if group is not None else 0
                dist.broadcast_object_list(obj, src=src, group=group)
                ctypes.memmove(buf, obj[0], NCCL_UNIQUE_ID_BYTES)
                _check(lib().xdit_comm_init(ctypes.cast(buf, _vp), n, rank, ulysses, ring, ctypes.byref(h)),
                       "xdit_comm_init")
            self.rank = rank
        self.handle = h
        self._reserved = None
        # per-channel message counters of mailbox users (PipeFusion stages, VAE bands): the device
        # flags keep their values across calls, so the tags must continue where the last call ended
        self.p2p_tags = {}

    def reserve(self, B: int, H: int, S_txt: int, S_img: int, D: int, elem_bytes: int = 2):
        """Collective when the shape changes (every rank, same scalars): reserve the workspace and,
        for the peer transport, exchange and map the peers' buffers."""
        key = (B, H, S_txt, S_img, D, elem_bytes)
        if self._reserved != key:
            peer = self.transport == "peer"
            if peer:  # nobody may still be writing into a buffer the reserve could reallocate
                import torch
                import torch.distributed as dist
                torch.cuda.synchronize()
                dist.barrier(group=self.group)
            _check(lib().xdit_comm_reserve(self.handle, *key), "xdit_comm_reserve")
            if peer:
                self.connect()
            self._reserved = key
        return self

    def connect(self):
        """Peer transport: export this rank's buffer descriptor, all-gather them, map the peers'."""
        import torch.distributed as dist
        blob = (ctypes.c_uint8 * PEER_BLOB_BYTES)()
        _check(lib().xdit_comm_peer_export(self.handle, ctypes.cast(blob, _vp)), "xdit_comm_peer_export")
        n = self.ulysses * self.ring
        blobs = [None] * n
        dist.all_gather_object(blobs, bytes(blob), group=self.group)
        allb = (ctypes.c_uint8 * (PEER_BLOB_BYTES * n)).from_buffer_copy(b"".join(blobs))
        _check(lib().xdit_comm_peer_connect(self.handle, ctypes.cast(allb, _vp)), "xdit_comm_peer_connect")

    # ---- peer-transport mailbox (point-to-point messages; see include/xdit_usp.h)
    def mailbox(self, bytes_per_src: int):
        """Collective: reserve >= bytes_per_src bytes of mailbox per source rank (re-connects)."""
        import torch
        import torch.distributed as dist
        if self.transport != "peer":
            raise XditError(1, "Comm.mailbox", "the mailbox needs the peer transport")
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        _check(lib().xdit_comm_mailbox_reserve(self.handle, int(bytes_per_src)), "xdit_comm_mailbox_reserve")
        self.connect()
        return self

    def mailbox_view(self, src: int, shape, dtype, offset: int = 0):
        """Torch view of this rank's mailbox region from rank `src` (no copy)."""
        import math
        import torch
        p, n = _vp(), ctypes.c_size_t()
        _check(lib().xdit_p2p_mailbox(self.handle, src, ctypes.byref(p), ctypes.byref(n)), "xdit_p2p_mailbox")
        esz = torch.empty((), dtype=dtype).element_size()
        if offset + math.prod(shape) * esz > n.value:
            raise XditError(9, "mailbox_view", "view exceeds the mailbox region")
        typestr = {torch.bfloat16: "<i2", torch.float32: "<f4", torch.float16: "<f2", torch.uint8: "|u1"}[dtype]

        class _Cai:
            __cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (p.value + offset, False),
                                        "version": 3, "strides": None}
        t = torch.as_tensor(_Cai(), device=torch.device("cuda", torch.cuda.current_device()))
        return t.view(dtype) if dtype == torch.bfloat16 else t

    def put(self, dst: int, src, tag: int, offset: int = 0, stream=None):
        n = src.numel() * src.element_size()
        _check(lib().xdit_p2p_put(self.handle, dst, _ptr(src), n, offset, tag & 0xFFFFFFFF, _stream(stream)),
               "xdit_p2p_put")

    def wait(self, src: int, tag: int, stream=None):
        _check(lib().xdit_p2p_wait(self.handle, src, tag & 0xFFFFFFFF, _stream(stream)), "xdit_p2p_wait")

    def ack(self, sender: int, tag: int, stream=None):
        _check(lib().xdit_p2p_ack(self.handle, sender, tag & 0xFFFFFFFF, _stream(stream)), "xdit_p2p_ack")

    def wait_ack(self, receiver: int, tag: int, stream=None):
        _check(lib().xdit_p2p_wait_ack(self.handle, receiver, tag & 0xFFFFFFFF, _stream(stream)), "xdit_p2p_wait_ack")

    def destroy(self):
        """Frees the handle.  Peer transport: every rank must have drained its streams first (the
        peers may still be writing into this rank's buffers) -- call collectively, after a barrier."""
        if self.handle:
            lib().xdit_comm_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.destroy()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def attention(q, k, v, *, S_txt: int, S_img: int, comm: Comm, ulysses: int = 1, ring: int = 1,
              out=None, lse=None, return_lse: bool = True, stream=None, kv_keep=None):
    """USP attention of this rank's local tokens: q, k, v [B, S_loc, H, D] (bf16 -> tcgen05 path,
    fp32 -> SIMT fp32 path).  Returns (out, lse) with lse [B, H, S_loc] fp32 (or None).
    kv_keep (bf16 only): a [2, B, H/ulysses, S_txt+S_img, D] bf16 CUDA tensor that receives the
    K,V of the whole SP group for this rank's heads (xdit_usp_attention_kv)."""
    import torch
    B, L, H, D = q.shape
    for t in (q, k, v):
        if not t.is_cuda or not t.is_contiguous():
            raise XditError(1, "attention", "q, k, v must be contiguous CUDA tensors")
    if out is None:
        out = torch.empty_like(q)
    if lse is None and return_lse:
        lse = torch.empty((B, H, L), dtype=torch.float32, device=q.device)
    f32 = q.dtype == torch.float32
    comm.reserve(B, H, S_txt, S_img, D, 4 if f32 else 2)
    if kv_keep is not None:
        if f32:
            raise XditError(2, "attention", "kv_keep is supported on the bf16 path only")
        rc = lib().xdit_usp_attention_kv(_ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), _ptr(kv_keep), B, H,
                                         S_txt, S_img, D, ulysses, ring, _stream(stream), comm.handle)
        _check(rc, "xdit_usp_attention_kv")
        return out, lse
    fn = lib().xdit_usp_attention_f32 if f32 else lib().xdit_usp_attention
    rc = fn(_ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), B, H, S_txt, S_img, D, ulysses, ring,
            _stream(stream), comm.handle)
    _check(rc, "xdit_usp_attention_f32" if f32 else "xdit_usp_attention")
    return out, lse


# ------------------------------------------------------------------------------------ stage kernels
def attn_scratch_bytes(D: int) -> int:
    return int(lib().xdit_attn_scratch_bytes(D))


def attn_fwd(q, k, v, o, lse, *, B: int, H: int, Sq: int, Skv: int, D: int, q_strides, kv_strides,
             omap: RowMap, dtype: int = 0, out_f32: int = 0, scratch=None, stream=None):
    """One attention launch (see xdit_attn_fwd).  Strides are (b, s, h) in elements.  `scratch`
    (a CUDA tensor of >= attn_scratch_bytes(D) bytes, or None) enables the tail split."""
    nbytes = 0 if scratch is None else scratch.numel() * scratch.element_size()
    rc = lib().xdit_attn_fwd(_ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), B, H, Sq, Skv, D,
                             *[int(x) for x in q_strides], *[int(x) for x in kv_strides],
                             ctypes.byref(omap), dtype, out_f32, _ptr(scratch), nbytes, _stream(stream))
    _check(rc, "xdit_attn_fwd")


def lse_merge(o_acc, lse_acc, o_s, lse_s, *, B: int, S: int, Hh: int, D: int, final=None,
              final_lse=None, final_map: Optional[RowMap] = None, final_dtype: int = 0, stream=None):
    rc = lib().xdit_lse_merge(_ptr(o_acc), _ptr(lse_acc), _ptr(o_s), _ptr(lse_s), B, S, Hh, D,
                              _ptr(final), _ptr(final_lse),
                              ctypes.byref(final_map) if final_map is not None else None,
                              final_dtype, _stream(stream))
    _check(rc, "xdit_lse_merge")


def uly_pack(x, send, *, B: int, L: int, Lmax: int, H: int, D: int, u: int, slot: int, nslots: int,
             elem_bytes: int, stream=None):
    _check(lib().xdit_uly_pack(_ptr(x), _ptr(send), B, L, Lmax, H, D, u, slot, nslots, elem_bytes,
                               _stream(stream)), "xdit_uly_pack")


def uly_unpack(recv, y, *, B: int, Lmax: int, Hh: int, D: int, u: int, lens, slot: int, nslots: int,
               elem_bytes: int, stream=None):
    arr = (_i * 8)(*([int(x) for x in lens] + [0] * (8 - len(lens))))
    _check(lib().xdit_uly_unpack(_ptr(recv), _ptr(y), B, Lmax, Hh, D, u, arr, slot, nslots, elem_bytes,
                                 _stream(stream)), "xdit_uly_unpack")


def uly_unpack_out(orecv_ptr: int, lrecv_ptr: Optional[int], peer_stride_bytes: int,
                   lse_peer_stride_bytes: int, out, lse, *, B: int, L: int, Lmax: int, Hh: int, D: int,
                   u: int, elem_bytes: int, stream=None):
    _check(lib().xdit_uly_unpack_out(orecv_ptr, lrecv_ptr, peer_stride_bytes, lse_peer_stride_bytes,
                                     _ptr(out), _ptr(lse), B, L, Lmax, Hh, D, u, elem_bytes,
                                     _stream(stream)), "xdit_uly_unpack_out")


# ------------------------------------------------------------------------- SURVEY §8(f) NEXT rows
def kv_retain(k_blk, v_blk, kv_keep, *, B: int, Hh: int, S_blk: int, S_total: int, seq_off: int, D: int,
              strides, stream=None):
    """Copy a K and a V block ([B][S_blk][Hh][D] with element strides (b, s, h)) into kv_keep
    [2][B][Hh][S_total][D] at rows [seq_off, seq_off + S_blk) (xdit_kv_retain)."""
    eb = k_blk.element_size()
    rc = lib().xdit_kv_retain(_ptr(k_blk), _ptr(v_blk), _ptr(kv_keep), B, Hh, S_blk, S_total, seq_off, D,
                              int(strides[0]), int(strides[1]), int(strides[2]), eb, _stream(stream))
    _check(rc, "xdit_kv_retain")


def cfg_combine(eps_cond, eps_uncond, g: float, out=None, stream=None):
    """eps_uncond + g (eps_cond - eps_uncond) on the GPU (fp32 math, one rounding to the dtype)."""
    import torch
    if out is None:
        out = torch.empty_like(eps_cond)
    dtype = 1 if eps_cond.dtype == torch.float32 else 0
    rc = lib().xdit_cfg_combine(_ptr(eps_cond), _ptr(eps_uncond), _ptr(out), eps_cond.numel(), float(g), dtype,
                                _stream(stream))
    _check(rc, "xdit_cfg_combine")
    return out


def cfg_tail(eps_local, g: float, *, comm: "Comm", gather=None, out=None, stream=None):
    """CFG step tail over a 2-rank handle: all-gather (rank 0 conditional, rank 1 unconditional),
    then the combine on every rank (xdit_cfg_tail)."""
    import torch
    n = eps_local.numel()
    if gather is None:
        gather = torch.empty((2,) + tuple(eps_local.shape), dtype=eps_local.dtype, device=eps_local.device)
    if out is None:
        out = torch.empty_like(eps_local)
    dtype = 1 if eps_local.dtype == torch.float32 else 0
    rc = lib().xdit_cfg_tail(_ptr(eps_local), _ptr(gather), _ptr(out), n, float(g), dtype, _stream(stream),
                             comm.handle)
    _check(rc, "xdit_cfg_tail")
    return out
