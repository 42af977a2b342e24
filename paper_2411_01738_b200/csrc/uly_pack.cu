// uly_pack.cu -- layout transforms around the Ulysses all-to-all.
// SP-Ulysses "employs All2All communications to transform the partitioning along the sequence
// dimension into partitioning along the head dimension" (§4.1.1).  Heads are split in
// contiguous blocks (reading C7); ragged shards are padded to Lmax in the exchange buffers and
// compacted on unpack (reading C5).  Pure data movement, HBM-bound: every kernel moves 16-byte (or
// narrower, if the row length demands) vectors with one thread per vector, so both the read and
// the write side are fully coalesced within each contiguous run.
#include <cuda_runtime.h>

#include <cstdint>

#include "xdit_internal.h"

namespace xdit {
namespace {

template <typename V>
__global__ void pack_kernel(const V* __restrict__ x, ChunkDst dst, int B, int L, int Lmax, int H, int Hh,
                            int vpr /* vectors per (row, head) */, int u, int slot, int nslots) {
  // x [B][L][H][vpr] -> chunk of Ulysses peer p = h / Hh: dst.p[p] [slot][B][Lmax][Hh][vpr].
  // dst.p[p] is this rank's send buffer at chunk p for the other Ulysses ranks, and its own receive
  // buffer at chunk j for its own head block (which therefore never crosses NCCL).
  const int64_t n = int64_t(B) * L * H * vpr;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int e = int(i % vpr);
    int64_t r = i / vpr;
    const int h = int(r % H);
    r /= H;
    const int l = int(r % L);
    const int b = int(r / L);
    const int p = h / Hh, hh = h - p * Hh;
    const int64_t chunk = int64_t(B) * Lmax * Hh * vpr;
    reinterpret_cast<V*>(dst.p[p])[int64_t(slot) * chunk + ((int64_t(b) * Lmax + l) * Hh + hh) * vpr + e] = x[i];
  }
}

template <typename V>
__global__ void unpack_kernel(const V* __restrict__ recv, V* __restrict__ y, int B, int Lmax,
                              int Hh, int vpr, int u, int4 len_lo, int4 len_hi, int S_blk,
                              int slot, int nslots) {
  // recv[p][slot][B][Lmax][Hh][vpr] -> y[B][S_blk][Hh][vpr], rows concatenated over p
  const int len[8] = {len_lo.x, len_lo.y, len_lo.z, len_lo.w, len_hi.x, len_hi.y, len_hi.z, len_hi.w};
  const int64_t n = int64_t(B) * S_blk * Hh * vpr;
  const int64_t chunk = int64_t(B) * Lmax * Hh * vpr;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int e = int(i % vpr);
    int64_t r = i / vpr;
    const int hh = int(r % Hh);
    r /= Hh;
    const int t = int(r % S_blk);
    const int b = int(r / S_blk);
    int p = 0, off = 0;
#pragma unroll
    for (int q = 0; q < 7; ++q)
      if (q + 1 < u && p == q && t >= off + len[q]) {  // segments are consecutive
        off += len[q];
        p = q + 1;
      }
    const int l = t - off;
    y[i] = recv[(int64_t(p) * nslots + slot) * chunk + ((int64_t(b) * Lmax + l) * Hh + hh) * vpr + e];
  }
}

template <typename V>
__global__ void unpack_out_kernel(const char* __restrict__ orecv, int64_t peer_stride, V* __restrict__ out,
                                  int B, int L, int Lmax, int Hh, int H, int vpr) {
  // orecv[p] (byte stride peer_stride) [B][Lmax][Hh][vpr] -> out[B][L][H][vpr], h = p*Hh + hh
  const int64_t n = int64_t(B) * L * H * vpr;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int e = int(i % vpr);
    int64_t r = i / vpr;
    const int h = int(r % H);
    r /= H;
    const int l = int(r % L);
    const int b = int(r / L);
    const int p = h / Hh, hh = h - p * Hh;
    const V* src = reinterpret_cast<const V*>(orecv + p * peer_stride);
    out[i] = src[((int64_t(b) * Lmax + l) * Hh + hh) * vpr + e];
  }
}

__global__ void unpack_lse_kernel(const char* __restrict__ lrecv, int64_t peer_stride,
                                  float* __restrict__ lse, int B, int L, int Lmax, int Hh, int H) {
  // lrecv[p] [B][Hh][Lmax] -> lse[B][H][L]
  const int64_t n = int64_t(B) * H * L;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int l = int(i % L);
    const int64_t bh = i / L;
    const int h = int(bh % H), b = int(bh / H);
    const int p = h / Hh, hh = h - p * Hh;
    const float* src = reinterpret_cast<const float*>(lrecv + p * peer_stride);
    lse[i] = src[(int64_t(b) * Hh + hh) * Lmax + l];
  }
}

unsigned grid_for(int64_t n, int threads) {
  int64_t g = (n + threads - 1) / threads;
  const int64_t cap = int64_t(device_sm_count()) * 16;
  return unsigned(g < 1 ? 1 : (g > cap ? cap : g));
}

int vec_bytes(int row_bytes) {
  if (row_bytes % 16 == 0) return 16;
  if (row_bytes % 8 == 0) return 8;
  if (row_bytes % 4 == 0) return 4;
  return 2;
}

}  // namespace

cudaError_t launch_uly_pack_to(const void* x, const ChunkDst& dst, int B, int L, int Lmax, int H, int D, int u,
                               int slot, int nslots, int elem_bytes, cudaStream_t st) {
  const int rb = D * elem_bytes, vb = vec_bytes(rb), vpr = rb / vb, Hh = H / u;
  const int64_t n = int64_t(B) * L * H * vpr;
  if (n == 0) return cudaSuccess;
  const unsigned g = grid_for(n, 256);
  switch (vb) {
    case 16: pack_kernel<uint4><<<g, 256, 0, st>>>((const uint4*)x, dst, B, L, Lmax, H, Hh, vpr, u, slot, nslots); break;
    case 8: pack_kernel<uint2><<<g, 256, 0, st>>>((const uint2*)x, dst, B, L, Lmax, H, Hh, vpr, u, slot, nslots); break;
    case 4: pack_kernel<uint32_t><<<g, 256, 0, st>>>((const uint32_t*)x, dst, B, L, Lmax, H, Hh, vpr, u, slot, nslots); break;
    default: pack_kernel<uint16_t><<<g, 256, 0, st>>>((const uint16_t*)x, dst, B, L, Lmax, H, Hh, vpr, u, slot, nslots); break;
  }
  note_launches(1);
  return cudaGetLastError();
}

cudaError_t launch_uly_pack(const void* x, void* send, int B, int L, int Lmax, int H, int D, int u,
                            int slot, int nslots, int elem_bytes, cudaStream_t st) {
  // send[p][slot][B][Lmax][H/u][D]: chunk p starts at p * nslots * (B * Lmax * H/u * D) elements
  ChunkDst dst{};
  const size_t chunk_bytes = size_t(nslots) * B * Lmax * (H / u) * D * elem_bytes;
  for (int p = 0; p < u && p < 8; ++p) dst.p[p] = static_cast<char*>(send) + p * chunk_bytes;
  return launch_uly_pack_to(x, dst, B, L, Lmax, H, D, u, slot, nslots, elem_bytes, st);
}

cudaError_t launch_uly_unpack(const void* recv, void* y, int B, int Lmax, int Hh, int D, int u,
                              const int* len, int slot, int nslots, int elem_bytes, cudaStream_t st) {
  int l8[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  int S_blk = 0;
  for (int p = 0; p < u; ++p) {
    l8[p] = len[p];
    S_blk += len[p];
  }
  const int4 lo = make_int4(l8[0], l8[1], l8[2], l8[3]), hi = make_int4(l8[4], l8[5], l8[6], l8[7]);
  const int rb = D * elem_bytes, vb = vec_bytes(rb), vpr = rb / vb;
  const int64_t n = int64_t(B) * S_blk * Hh * vpr;
  if (n == 0) return cudaSuccess;
  const unsigned g = grid_for(n, 256);
  switch (vb) {
    case 16: unpack_kernel<uint4><<<g, 256, 0, st>>>((const uint4*)recv, (uint4*)y, B, Lmax, Hh, vpr, u, lo, hi, S_blk, slot, nslots); note_launches(1); break;
    case 8: unpack_kernel<uint2><<<g, 256, 0, st>>>((const uint2*)recv, (uint2*)y, B, Lmax, Hh, vpr, u, lo, hi, S_blk, slot, nslots); note_launches(1); break;
    case 4: unpack_kernel<uint32_t><<<g, 256, 0, st>>>((const uint32_t*)recv, (uint32_t*)y, B, Lmax, Hh, vpr, u, lo, hi, S_blk, slot, nslots); note_launches(1); break;
    default: unpack_kernel<uint16_t><<<g, 256, 0, st>>>((const uint16_t*)recv, (uint16_t*)y, B, Lmax, Hh, vpr, u, lo, hi, S_blk, slot, nslots); note_launches(1); break;
  }
  return cudaGetLastError();
}

cudaError_t launch_uly_unpack_out(const void* orecv, const float* lrecv, int64_t peer_stride_bytes,
                                  int64_t lse_peer_stride_bytes, void* out, float* lse, int B, int L,
                                  int Lmax, int Hh, int D, int u, int elem_bytes, cudaStream_t st) {
  const int H = Hh * u;
  const int rb = D * elem_bytes, vb = vec_bytes(rb), vpr = rb / vb;
  const int64_t n = int64_t(B) * L * H * vpr;
  if (n > 0) {
    const unsigned g = grid_for(n, 256);
    const char* src = static_cast<const char*>(orecv);
    switch (vb) {
      case 16: unpack_out_kernel<uint4><<<g, 256, 0, st>>>(src, peer_stride_bytes, (uint4*)out, B, L, Lmax, Hh, H, vpr); note_launches(1); break;
      case 8: unpack_out_kernel<uint2><<<g, 256, 0, st>>>(src, peer_stride_bytes, (uint2*)out, B, L, Lmax, Hh, H, vpr); note_launches(1); break;
      case 4: unpack_out_kernel<uint32_t><<<g, 256, 0, st>>>(src, peer_stride_bytes, (uint32_t*)out, B, L, Lmax, Hh, H, vpr); note_launches(1); break;
      default: unpack_out_kernel<uint16_t><<<g, 256, 0, st>>>(src, peer_stride_bytes, (uint16_t*)out, B, L, Lmax, Hh, H, vpr); note_launches(1); break;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  if (lse && lrecv && int64_t(B) * H * L > 0) {
    unpack_lse_kernel<<<grid_for(int64_t(B) * H * L, 256), 256, 0, st>>>(
        reinterpret_cast<const char*>(lrecv), lse_peer_stride_bytes, lse, B, L, Lmax, Hh, H); note_launches(1);
  }
  return cudaGetLastError();
}

}  // namespace xdit
