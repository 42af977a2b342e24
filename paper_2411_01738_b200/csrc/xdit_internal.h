// xdit_internal.h -- declarations shared by the host orchestrator (xdit_usp.cpp) and the CUDA
// kernel launchers.  Not part of the public ABI (that is include/xdit_usp.h).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/xdit_usp.h"

namespace xdit {

// Count one kernel launch of this library (xdit_launch_count()).
void note_launches(int n);

// SM count of the CURRENT device (cached per device ordinal: a process may drive several GPUs).
int device_sm_count();

// One flag per device ordinal (e.g. "cudaFuncSetAttribute done for this kernel on device d").
struct DeviceFlags {
  unsigned long long bits[2] = {0, 0};  // devices 0..127
  static int cur() {
    int d = 0;
    cudaGetDevice(&d);
    return d & 127;
  }
  bool test() const {
    const int d = cur();
    return (__atomic_load_n(&bits[d >> 6], __ATOMIC_ACQUIRE) >> (d & 63)) & 1ull;
  }
  void set() {
    const int d = cur();
    __atomic_fetch_or(&bits[d >> 6], 1ull << (d & 63), __ATOMIC_RELEASE);
  }
};

// Arguments of one attention launch (one Q block against one KV block).  Strides in elements.
struct AttnArgs {
  const void* q;
  const void* k;
  const void* v;
  void* o;
  float* lse;  // may be null
  int B, H, Sq, Skv, D;
  int64_t q_b, q_s, q_h;
  int64_t kv_b, kv_s, kv_h;
  xdit_rowmap omap;
  int out_f32;
  float* scratch = nullptr;    // optional fp32 scratch for the tail split (bf16 kernel), may be null
  size_t scratch_floats = 0;
  // ring merge fused into the epilogue (see EpiParams in attn_common.cuh); only where
  // attn_fused_merge_supported() says so
  int merge = 0, merge_final = 0;
  float* acc_o = nullptr;
  const float* acc_l_in = nullptr;
  float* acc_l_out = nullptr;
  xdit_rowmap acc_map{};
};
// True when launch_attn_fwd_bf16 runs a kernel that implements the fused ring merge.
bool attn_fused_merge_supported(int D);

// fp32 scratch the bf16 attention kernel can use to split the last partial wave of its grid:
// (#SMs) x 256 rows x (D + 1) floats.
size_t attn_scratch_floats(int D);

// Launchers return cudaError_t (cudaSuccess on success); argument checks happen in xdit_usp.cpp.
// bf16, D in {64,72,128}: the CTA-pair (cta_group::2) tcgen05 kernel (attn_fwd_2sm.cu)
cudaError_t launch_attn_fwd_bf16(const AttnArgs& a, cudaStream_t st);
cudaError_t launch_attn_fwd_f32(const AttnArgs& a, cudaStream_t st);    // fp32 SIMT, D <= 256
cudaError_t launch_lse_merge(float* o_acc, float* lse_acc, const float* o_s, const float* lse_s,
                             int B, int S, int Hh, int D, void* fin, float* fin_lse,
                             const xdit_rowmap* fmap, int fin_dtype, cudaStream_t st);
// Per-Ulysses-peer destination base addresses of a pack (the send chunk of each peer; this rank's
// own head block goes straight to its receive chunk).
struct ChunkDst {
  char* p[8];
};
cudaError_t launch_uly_pack_to(const void* x, const ChunkDst& dst, int B, int L, int Lmax, int H, int D, int u,
                               int slot, int nslots, int elem_bytes, cudaStream_t st);
cudaError_t launch_uly_pack(const void* x, void* send, int B, int L, int Lmax, int H, int D, int u,
                            int slot, int nslots, int elem_bytes, cudaStream_t st);
cudaError_t launch_uly_unpack(const void* recv, void* y, int B, int Lmax, int Hh, int D, int u,
                              const int* len, int slot, int nslots, int elem_bytes,
                              cudaStream_t st);
cudaError_t launch_uly_unpack_out(const void* orecv, const float* lrecv, int64_t peer_stride_bytes,
                                  int64_t lse_peer_stride_bytes, void* out, float* lse, int B,
                                  int L, int Lmax, int Hh, int D, int u, int elem_bytes,
                                  cudaStream_t st);

// SURVEY §8(f) NEXT rows (next_ops.cu).
// Where the rows of a K/V block land in a KV buffer: block rows [src[k], src[k+1]) (src[n] = the
// block's row count) go to buffer rows dst[k] + (t - src[k]).
struct KvSegs {
  int n;
  int src[16], dst[16];
};
cudaError_t launch_kv_place(const void* k, const void* v, void* kv, int B, int Hh, int S_blk, int S_total,
                            const KvSegs& segs, int D, int64_t sb, int64_t ss, int64_t sh, int eb, cudaStream_t st);
cudaError_t launch_kv_retain(const void* k, const void* v, void* kv_keep, int B, int Hh, int S_blk, int S_total,
                             int seq_off, int D, int64_t sb, int64_t ss, int64_t sh, int eb, cudaStream_t st);
cudaError_t launch_cfg_combine(const void* c, const void* u, void* o, int64_t n, float g, int dtype,
                               cudaStream_t st);

// SURVEY §8(f) NEXT 3, PipeFusion on a synthetic DiT stack (pipefusion.cu).
size_t pf_workspace_bytes(int B, int n, int H, int D, int dtype);
cudaError_t launch_pf_block(void* h, void* kv, const float* w, void* work, int B, int H, int S, int off, int n,
                            int D, int dtype, cudaStream_t st);
cudaError_t launch_pf_sampler(void* x, const void* eps, int64_t n, float sigma, int dtype, cudaStream_t st);
cudaError_t launch_pf_qkv(const void* h, const float* w, void* q, void* k, void* v, int B, int n, int H, int D,
                          int dtype, cudaStream_t st);
cudaError_t launch_pf_residual(void* h, const void* o, const float* w, int B, int n, int H, int D, int dtype,
                               cudaStream_t st);

// SURVEY §8(f) NEXT 4, patch-parallel VAE decode (vae.cu).
cudaError_t launch_vae_conv3x3(const float* in, int Hout, int Ci, int W, const float* w, const float* b, float* out,
                               int Co, int act_up, cudaStream_t st);
cudaError_t launch_vae_conv_tc(const void* in, int Hout, int Ci, int W, const void* wt, const float* b, void* out,
                               int Co, int act_up, cudaStream_t st);

// Device-side row-map resolution shared by every epilogue that writes through an xdit_rowmap.
struct RowDst {
  int64_t o_off;  // element offset of (b, row, h, 0)
  int64_t l_off;  // element offset of lse(b, h, row)
};
__host__ __device__ inline RowDst rowmap_dst(const xdit_rowmap& m, int b, int row, int h) {
  int s = 0;
#if defined(__CUDACC__)
#pragma unroll
#endif
  for (int i = 1; i < 8; ++i)
    if (i < m.nseg && row >= m.seg_off[i]) s = i;
  const int64_t r = row - m.seg_off[s];
  RowDst d;
  d.o_off = s * m.o_seg + b * m.o_b + r * m.o_s + h * m.o_h;
  d.l_off = s * m.l_seg + b * m.l_b + h * m.l_h + r;
  return d;
}

}  // namespace xdit
