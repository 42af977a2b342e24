"""fp64 CPU oracle for the USP attention hot path (arXiv 2411.01738) -- TEST INFRASTRUCTURE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product package ``paper_2411_01738_b200``
never imports it, and the two share no code: this is a ctypes wrapper around ``xdit_oracle.c``
(plain C, fp64) whose header cites the PAPER.md passage each function follows.

Functions (numpy float64 arrays, layouts as in xdit_oracle.c):
  attention(q, k, v)            -> out [B,Sq,H,D], lse [B,H,Sq]      (P:257 full attention; C1/C2)
  attention_rows(q, k, v, rows) -> out [B,n,H,D],  lse [B,H,n]       (exact subset of the above)
  shard(S_txt, S_img, N, g)     -> (txt_off, txt_len, img_off, img_len)   (reading C5)
  usp_emulate(q, k, v, S_txt, u, r) -> out, lse                      (readings C5-C9)
  kv_keep(k, v, S_txt, u, r, g) -> [2,B,H/u,S,D]  KV buffer rank g retains (NEXT 1)
  cfg_combine(eps_cond, eps_uncond, g) -> eps_uncond + g (eps_cond - eps_uncond)  (NEXT 2)
  pipefusion.*  (submodule, numpy fp64): PipeFusion on a synthetic DiT stack -- patch bounds, the
                staleness replay and the stale-KV numerics (NEXT 3, reading R4)
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "xdit_oracle.c")
_LIB_PATH = os.path.join(_HERE, "libxdit_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (IEEE fp64: no fast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-ffp-contract=off", "-fno-fast-math",
               "-Wall", "-o", _LIB_PATH, _SRC, "-lm", "-lpthread"]
        subprocess.check_call(cmd)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB_PATH)
        dp = ctypes.POINTER(ctypes.c_double)
        ip = ctypes.POINTER(ctypes.c_int)
        i64p = ctypes.POINTER(ctypes.c_int64)
        c_int, c_double = ctypes.c_int, ctypes.c_double
        lib.xo_attention.argtypes = [dp, dp, dp, dp, dp, c_int, c_int, c_int, c_int, c_int, c_double, c_int]
        lib.xo_attention.restype = c_int
        lib.xo_attention_rows.argtypes = [dp, dp, dp, i64p, c_int, dp, dp, c_int, c_int, c_int, c_int,
                                          c_int, c_double, c_int]
        lib.xo_attention_rows.restype = c_int
        lib.xo_shard.argtypes = [c_int, c_int, c_int, c_int, ip, ip, ip, ip]
        lib.xo_shard.restype = c_int
        lib.xo_usp_emulate.argtypes = [dp, dp, dp, dp, dp, c_int, c_int, c_int, c_int, c_int, c_int, c_int]
        lib.xo_usp_emulate.restype = c_int
        lib.xo_default_threads.argtypes = []
        lib.xo_default_threads.restype = c_int
        _lib = lib
    return _lib


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def default_threads() -> int:
    return int(_load().xo_default_threads())


def attention(q, k, v, scale: float = 0.0, nthreads: int = 0):
    """Plain fp64 softmax(q k^T * scale) v over [B,S,H,D]; scale<=0 means 1/sqrt(D)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    B, Sq, H, D = q.shape
    Skv = k.shape[1]
    assert k.shape == (B, Skv, H, D) and v.shape == (B, Skv, H, D)
    out = np.empty((B, Sq, H, D), np.float64)
    lse = np.empty((B, H, Sq), np.float64)
    rc = _load().xo_attention(_p(q), _p(k), _p(v), _p(out), _p(lse), B, Sq, Skv, H, D, float(scale),
                              int(nthreads))
    if rc != 0:
        raise ValueError(f"xo_attention failed rc={rc}")
    return out, lse


def attention_rows(q, k, v, rows, scale: float = 0.0, nthreads: int = 0):
    """fp64 attention for the given global query rows only (exact subset of ``attention``)."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    rows = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
    B, Sq, H, D = q.shape
    Skv = k.shape[1]
    n = int(rows.size)
    out = np.empty((B, n, H, D), np.float64)
    lse = np.empty((B, H, n), np.float64)
    rc = _load().xo_attention_rows(_p(q), _p(k), _p(v), rows.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                   n, _p(out), _p(lse), B, Sq, Skv, H, D, float(scale), int(nthreads))
    if rc != 0:
        raise ValueError(f"xo_attention_rows failed rc={rc}")
    return out, lse


def shard(S_txt: int, S_img: int, N: int, g: int):
    """(txt_off, txt_len, img_off, img_len) of rank g; raises on an empty shard."""
    vals = [ctypes.c_int() for _ in range(4)]
    rc = _load().xo_shard(S_txt, S_img, N, g, *[ctypes.byref(x) for x in vals])
    if rc != 0:
        raise ValueError(f"xo_shard rc={rc}")
    return tuple(int(x.value) for x in vals)


def local_rows(S_txt: int, S_img: int, N: int, g: int) -> np.ndarray:
    """Global joint-sequence rows ([text; image], reading C4) held by rank g, in local order."""
    to, tl, io, il = shard(S_txt, S_img, N, g)
    return np.concatenate([np.arange(to, to + tl), S_txt + np.arange(io, io + il)]).astype(np.int64)


def usp_emulate(q, k, v, S_txt: int, u: int, r: int):
    """fp64 step-by-step emulation of USP (Ulysses u x Ring r) on global [B,S,H,D] tensors."""
    q, k, v = _f64(q), _f64(k), _f64(v)
    B, S, H, D = q.shape
    out = np.full((B, S, H, D), np.nan)
    lse = np.full((B, H, S), np.nan)
    rc = _load().xo_usp_emulate(_p(q), _p(k), _p(v), _p(out), _p(lse), B, H, S_txt, S - S_txt, D, u, r)
    if rc != 0:
        raise ValueError(f"xo_usp_emulate failed rc={rc}")
    return out, lse


def kv_keep(k, v, S_txt: int, u: int, r: int, g: int) -> np.ndarray:
    """The KV buffer rank g of a USP (Ulysses u x Ring r) group retains after one attention call --
    SURVEY §8(f) NEXT 1, PAPER P:401-407 ("after communication of K and V in SP-Ulysses and SP-Ring,
    the intermediate results ... are stored in each device's KV Buffer"; "For SP-Ulysses, we obtain
    the KV of the sequence within the SP group participating in the computation of the head ... For
    SP-Ring, we obtain the KV of the sequence within the SP group for all heads").

    Reading (DESIGN.md §3 R2): with USP the rank holds, for its Ulysses head block j = g mod u
    (heads [j H/u, (j+1) H/u), reading C7), the K and V of EVERY token of the SP group -- the
    all-to-all gathers its ring block's tokens and the ring rotation brings the other r-1 blocks --
    laid out [2 (K, V)][B][H/u][S][D] with the sequence in SP-shard order: rank 0's local rows, then
    rank 1's, ... (each rank's local rows = its text shard then its image shard, reading C5).
    Index math only: k, v are the global [B, S, H, D] tensors."""
    k, v = np.asarray(k), np.asarray(v)
    B, S, H, D = k.shape
    N, j, Hh = u * r, g % u, H // u
    rows = np.concatenate([local_rows(S_txt, S - S_txt, N, p) for p in range(N)])
    out = np.empty((2, B, Hh, S, D), dtype=k.dtype)
    for t, x in enumerate((k, v)):
        out[t] = x[:, rows][:, :, j * Hh:(j + 1) * Hh].transpose(0, 2, 1, 3)
    return out


def cfg_combine(eps_cond, eps_uncond, g: float) -> np.ndarray:
    """Classifier-free-guidance combine of the two CFG branches' noise predictions, computed in fp64
    -- SURVEY §8(f) NEXT 2 (the two latents are computed separately and gathered
    after each step; eps_uncond + g (eps_cond - eps_uncond))."""
    c, u_ = _f64(eps_cond), _f64(eps_uncond)
    assert c.shape == u_.shape
    return u_ + float(g) * (c - u_)
