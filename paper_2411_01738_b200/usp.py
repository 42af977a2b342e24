"""Thin ctypes binding of libxdit_usp.so (include/xdit_usp.h).

Argument marshalling only: torch tensors -> device pointers, the current CUDA stream -> handle,
status codes -> exceptions.  Every step of the hot path runs in the library's CUDA kernels and
NCCL; there is no Python or CPU fallback -- if the extension is missing this module raises.
The binding refuses a library whose xdit_version() differs from ABI_VERSION (the struct layouts
below are those of include/xdit_usp.h at that version).
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence, Tuple

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libxdit_usp.so")
# Same-session kernel A/Bs (tools/ab_attn.sh) load a tagged build of this same source,
# paper_2411_01738_b200/libxdit_usp_<tag>.so (python -m paper_2411_01738_b200.build --tag=...), by
# XDIT_LIB; nothing else is accepted.
_ab = os.environ.get("XDIT_LIB")
if _ab:
    _ab = os.path.abspath(_ab)
    if os.path.dirname(_ab) != HERE or not os.path.basename(_ab).startswith("libxdit_usp_"):
        raise ImportError(f"XDIT_LIB={_ab}: only tagged builds paper_2411_01738_b200/libxdit_usp_<tag>.so")
    LIB_PATH = _ab

ABI_VERSION = 30000  # XDIT_ABI_VERSION of include/xdit_usp.h
XDIT_STATUS = {0: "OK", 1: "INVALID_ARG", 2: "UNSUPPORTED", 3: "DIVISIBILITY", 4: "COMM_MISMATCH",
               5: "EMPTY_SHARD", 6: "ALIGNMENT", 7: "CUDA", 8: "NCCL", 9: "WORKSPACE"}
NCCL_UNIQUE_ID_BYTES = 128


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
                ("l_h", ctypes.c_int64)]

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


class P2POp(ctypes.Structure):
    """xdit_p2p_op: one send or receive of an xdit_p2p group."""
    _fields_ = [("peer", ctypes.c_int32), ("is_send", ctypes.c_int32), ("buf", ctypes.c_void_p),
                ("bytes", ctypes.c_size_t)]


class Phases(ctypes.Structure):
    """xdit_phases: per-phase timing of the last profiled xdit_usp_attention call."""
    _fields_ = [("valid", ctypes.c_int32), ("ulysses", ctypes.c_int32), ("ring", ctypes.c_int32),
                ("pad_", ctypes.c_int32), ("total_ms", ctypes.c_float), ("a2a_in_ms", ctypes.c_float),
                ("a2a_out_ms", ctypes.c_float), ("pad2_", ctypes.c_float), ("attn_ms", ctypes.c_float * 8),
                ("ring_comm_ms", ctypes.c_float * 8), ("a2a_in_bytes", ctypes.c_int64),
                ("a2a_out_bytes", ctypes.c_int64), ("ring_bytes", ctypes.c_int64 * 8)]

    def as_dict(self):
        r = self.ring
        return {"total_ms": self.total_ms, "a2a_in_ms": self.a2a_in_ms, "a2a_out_ms": self.a2a_out_ms,
                "attn_ms": list(self.attn_ms[:r]), "ring_comm_ms": list(self.ring_comm_ms[:max(0, r - 1)]),
                "a2a_in_bytes": int(self.a2a_in_bytes), "a2a_out_bytes": int(self.a2a_out_bytes),
                "ring_bytes": [int(x) for x in self.ring_bytes[:max(0, r - 1)]]}


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
    "xdit_p2p": ([_vp, ctypes.POINTER(P2POp), _i, _vp], _i),
    "xdit_comm_profile": ([_vp, _i], _i),
    "xdit_comm_phases": ([_vp, ctypes.POINTER(Phases)], _i),
    "xdit_comm_reserve": ([_vp, _i, _i, _i, _i, _i, _i], _i),
    "xdit_comm_info": ([_vp] + [ctypes.POINTER(_i)] * 4, _i),
    "xdit_comm_destroy": ([_vp], _i),
    "xdit_usp_attention": ([_vp] * 5 + [_i] * 7 + [_vp, _vp], _i),
    "xdit_usp_attention_f32": ([_vp] * 5 + [_i] * 7 + [_vp, _vp], _i),
    "xdit_usp_attention_kv": ([_vp] * 6 + [_i] * 7 + [_vp, _vp], _i),
    "xdit_usp_attention_buf": ([_vp] * 6 + [_i] * 11 + [_vp, _vp], _i),
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
    "xdit_pf_qkv": ([_vp] * 5 + [_i] * 5 + [_vp], _i),
    "xdit_pf_residual": ([_vp] * 3 + [_i] * 5 + [_vp], _i),
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
        if L.xdit_version() != ABI_VERSION:
            raise ImportError(f"{LIB_PATH} has ABI {L.xdit_version()}, this binding needs {ABI_VERSION}: rebuild it")
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


def _torch_nccl_comm(group):
    """The ncclComm_t of a torch ProcessGroupNCCL (its `_comm_ptr()`), or None for another backend.
    torch creates a group's communicator lazily; a 1-element all_reduce forces it into existence."""
    import torch
    import torch.distributed as dist
    pg = group if group is not None else dist.distributed_c10d._get_default_group()
    if dist.get_backend(pg) != "nccl":
        return None
    be = pg._get_backend(torch.device("cuda", torch.cuda.current_device()))
    ptr = be._comm_ptr() if hasattr(be, "_comm_ptr") else 0
    if not ptr:
        t = torch.zeros(1, device="cuda")
        dist.all_reduce(t, group=pg)
        torch.cuda.synchronize()
        ptr = be._comm_ptr()
    return int(ptr) or None


class Comm:
    """One SP group (= one CFG group): ulysses x ring mesh, NCCL communicators, workspace.

    Every byte between ranks moves over NCCL.  If `group` (torch.distributed, default: the world) is
    an NCCL process group, the handle splits that group's own communicator (`pg._comm_ptr()` ->
    xdit_comm_create); otherwise (e.g. a gloo group carrying only host plumbing) rank
    0 creates an NCCL unique id, torch.distributed broadcasts it and every rank calls
    xdit_comm_init.  With ulysses*ring == 1 no communicator is made."""

    def __init__(self, ulysses: int = 1, ring: int = 1, group=None):
        self.ulysses, self.ring, self.group = ulysses, ring, group
        n = ulysses * ring
        h = _vp()
        self.source = None
        if n == 1:
            _check(lib().xdit_comm_init(None, 1, 0, 1, 1, ctypes.byref(h)), "xdit_comm_init")
            self.rank = 0
        else:
            import torch.distributed as dist
            rank = dist.get_rank(group)
            if dist.get_world_size(group) != n:
                raise XditError(4, "Comm", f"group size {dist.get_world_size(group)} != ulysses*ring={n}")
            ptr = _torch_nccl_comm(group)
            if ptr is not None:
                _check(lib().xdit_comm_create(ptr, ulysses, ring, ctypes.byref(h)), "xdit_comm_create")
                self.source = "torch ProcessGroupNCCL._comm_ptr()"
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
                self.source = "own NCCL communicator (unique id over torch.distributed)"
            self.rank = rank
        self.handle = h
        self._reserved = None

    @property
    def size(self) -> int:
        return self.ulysses * self.ring

    def reserve(self, B: int, H: int, S_txt: int, S_img: int, D: int, elem_bytes: int = 2):
        """Workspace for a shape (every rank, same scalars; a no-op when it already fits)."""
        key = (B, H, S_txt, S_img, D, elem_bytes)
        if self._reserved != key:
            _check(lib().xdit_comm_reserve(self.handle, *key), "xdit_comm_reserve")
            self._reserved = key
        return self

    def p2p(self, ops, stream=None):
        """One NCCL group of sends / receives: ops = [(peer, "send" | "recv", tensor), ...]
        (xdit_p2p; contiguous CUDA tensors, the receiving side's tensor has the same byte size)."""
        arr = (P2POp * max(1, len(ops)))()
        for x, (peer, kind, t) in enumerate(ops):
            if kind not in ("send", "recv"):
                raise XditError(1, "Comm.p2p", f"op kind must be 'send' or 'recv', got {kind!r}")
            if not t.is_contiguous():
                raise XditError(1, "Comm.p2p", "tensors must be contiguous")
            arr[x] = P2POp(int(peer), 1 if kind == "send" else 0, _ptr(t), t.numel() * t.element_size())
        _check(lib().xdit_p2p(self.handle, arr, len(ops), _stream(stream)), "xdit_p2p")

    def profile(self, enable: bool = True):
        """Record per-phase timing events in the following calls (xdit_comm_profile)."""
        _check(lib().xdit_comm_profile(self.handle, 1 if enable else 0), "xdit_comm_profile")

    def phases(self) -> Optional[dict]:
        """Per-phase times and bytes of the last profiled call (host-synchronising), or None."""
        ph = Phases()
        _check(lib().xdit_comm_phases(self.handle, ctypes.byref(ph)), "xdit_comm_phases")
        return ph.as_dict() if ph.valid else None

    def destroy(self):
        """Frees the handle (device-synchronising; collective only in that peers must have finished
        the calls they share with this rank)."""
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


def attention_buf(q, k, v, kv_buf, *, S_txt: int, S_img: int, txt_row: int, img_row: int, comm: Comm,
                  ulysses: int = 1, ring: int = 1, out=None, lse=None, stream=None):
    """USP attention of one PipeFusion patch over the persistent KV buffer (xdit_usp_attention_buf,
    hybrid PipeFusion x SP, NEXT 3): q, k, v this rank's rows of the patch [B, S_loc, H, D] (the
    patch = S_txt text + S_img image tokens); kv_buf [2, B, H/ulysses, S_buf, D] of the same dtype,
    the patch's text token t at row txt_row + t, image token t at img_row + t.  Returns (out, lse)."""
    import torch
    B, L, H, D = q.shape
    for t in (q, k, v, kv_buf):
        if not t.is_cuda or not t.is_contiguous():
            raise XditError(1, "attention_buf", "q, k, v, kv_buf must be contiguous CUDA tensors")
    if out is None:
        out = torch.empty_like(q)
    f32 = q.dtype == torch.float32
    comm.reserve(B, H, S_txt, S_img, D, 4 if f32 else 2)
    S_buf = kv_buf.shape[3]
    rc = lib().xdit_usp_attention_buf(_ptr(q), _ptr(k), _ptr(v), _ptr(out), _ptr(lse), _ptr(kv_buf), B, H, S_txt,
                                      S_img, D, ulysses, ring, S_buf, txt_row, img_row, 1 if f32 else 0,
                                      _stream(stream), comm.handle)
    _check(rc, "xdit_usp_attention_buf")
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
