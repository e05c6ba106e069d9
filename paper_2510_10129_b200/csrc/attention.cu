// Legacy (mma.sync) sparse-row attention — the round-1 baseline.
//
// sparse_row_attention_kernel — causal_attention(..., row_limits=idx+1)
//     of selective_forward (model.py:715-720) and the mask_offset rule of
//     layer_forward (model.py:467-476), without materialising the (H, m, n)
//     logits (tensor_core.py:166-170). Flash-style online softmax over a bf16
//     bank; GQA packing puts the G query heads of one KV head on the same
//     64-row tile so every K/V tile is loaded once for all of them; each tile
//     streams keys only up to its largest row limit (selected rows are sorted,
//     so a tile spans a narrow position range). Round-1 version on
//     mma.sync.m16n8k16 (bf16 -> fp32).
//
// The tcgen05 kernel that replaced it for production is attention_sm100.cu;
// this one stays as the measured legacy-tensor-core baseline.
#include "cc_common.cuh"

namespace cc {

// ---------------------------------------------------------------------------
// (1) bf16 sparse-row flash attention
// ---------------------------------------------------------------------------
constexpr int kAttnRows = 64;   // packed query rows per CTA (4 warps x 16)
constexpr int kAttnKeys = 64;   // keys per smem tile
constexpr int kAttnThreads = 128;

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int n = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(n) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma_bf16(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int HD>
__global__ void __launch_bounds__(kAttnThreads) sparse_row_attention_kernel(
    const __nv_bfloat16* __restrict__ q, int64_t ldq, const int64_t* __restrict__ pos, int64_t m,
    const __nv_bfloat16* __restrict__ kc, const __nv_bfloat16* __restrict__ vc, int64_t n_keys, int n_q_heads,
    int n_kv_heads, float factor, const float* __restrict__ row_factor, __nv_bfloat16* __restrict__ out,
    int64_t ldo) {
  constexpr int CH = HD / 8;            // 16-byte chunks per key row
  constexpr int ROWB = HD * 2;          // bytes per key row
  constexpr int TILEB = kAttnKeys * ROWB;
  extern __shared__ __align__(128) uint8_t smem[];
  // [K0][V0][K1][V1]
  __shared__ int s_lim_max;

  const int G = n_q_heads / n_kv_heads;
  const int kvh = blockIdx.y;
  const int64_t packed_total = m * G;
  const int64_t p_base = (int64_t)blockIdx.x * kAttnRows;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const float LOG2E = 1.4426950408889634f;

  // this thread's two rows (g, g+8) of the warp's 16
  int64_t prow[2];
  int lim[2];
  float scale2[2];
  const __nv_bfloat16* qrow[2];
  int64_t orow_off[2];
  bool valid[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int64_t p = p_base + warp * 16 + g + h * 8;
    prow[h] = p;
    valid[h] = p < packed_total;
    const int64_t i = valid[h] ? p / G : 0;
    const int head = kvh * G + (valid[h] ? (int)(p % G) : 0);
    const int64_t ps = valid[h] ? pos[i] : -1;
    const int64_t l = ps + 1 < n_keys ? ps + 1 : n_keys;
    lim[h] = (int)l;
    const float f = row_factor ? (valid[h] ? row_factor[i] : 0.f) : factor;
    scale2[h] = f * LOG2E;
    qrow[h] = q + i * ldq + (int64_t)head * HD;
    orow_off[h] = i * ldo + (int64_t)head * HD;
  }
  // CTA-wide maximum key limit
  if (threadIdx.x == 0) s_lim_max = 0;
  __syncthreads();
  int my_max = max(lim[0], lim[1]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) my_max = max(my_max, __shfl_xor_sync(0xffffffffu, my_max, o));
  if (lane == 0) atomicMax(&s_lim_max, my_max);
  __syncthreads();
  const int kmax = s_lim_max;
  const int n_tiles = (kmax + kAttnKeys - 1) / kAttnKeys;
  int warp_min = min(valid[0] ? lim[0] : 1 << 30, valid[1] ? lim[1] : 1 << 30);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) warp_min = min(warp_min, __shfl_xor_sync(0xffffffffu, warp_min, o));

  // Q fragments (A operand, 16 rows x HD)
  uint32_t qf[HD / 16][4];
#pragma unroll
  for (int kk = 0; kk < HD / 16; ++kk) {
    const int c = kk * 16 + 2 * t;
    qf[kk][0] = valid[0] ? *reinterpret_cast<const uint32_t*>(qrow[0] + c) : 0u;
    qf[kk][1] = valid[1] ? *reinterpret_cast<const uint32_t*>(qrow[1] + c) : 0u;
    qf[kk][2] = valid[0] ? *reinterpret_cast<const uint32_t*>(qrow[0] + c + 8) : 0u;
    qf[kk][3] = valid[1] ? *reinterpret_cast<const uint32_t*>(qrow[1] + c + 8) : 0u;
  }

  float o_acc[HD / 8][4];
#pragma unroll
  for (int i = 0; i < HD / 8; ++i) o_acc[i][0] = o_acc[i][1] = o_acc[i][2] = o_acc[i][3] = 0.f;
  float row_m[2] = {-INFINITY, -INFINITY}, row_l[2] = {0.f, 0.f};

  const uint32_t sbase = smem_u32(smem);
  const int64_t kv_stride = (int64_t)n_kv_heads * HD;
  auto load_tile = [&](int tile, int buf) {
    const uint32_t kdst = sbase + buf * 2 * TILEB;
    const uint32_t vdst = kdst + TILEB;
    for (int idx = threadIdx.x; idx < kAttnKeys * CH; idx += kAttnThreads) {
      const int r = idx / CH, c = idx % CH;
      const int64_t key = (int64_t)tile * kAttnKeys + r;
      const bool ok = key < n_keys;
      const int64_t off = (ok ? key : 0) * kv_stride + (int64_t)kvh * HD + c * 8;
      const uint32_t soff = r * ROWB + ((c ^ (r & 7)) * 16);
      cp_async16(kdst + soff, kc + off, ok);
      cp_async16(vdst + soff, vc + off, ok);
    }
    cp_async_commit();
  };

  if (n_tiles > 0) load_tile(0, 0);
  for (int tile = 0; tile < n_tiles; ++tile) {
    const int buf = tile & 1;
    if (tile + 1 < n_tiles) {
      load_tile(tile + 1, buf ^ 1);
      cp_async_wait<1>();
    } else {
      cp_async_wait<0>();
    }
    __syncthreads();
    const uint32_t ks = sbase + buf * 2 * TILEB;
    const uint32_t vs = ks + TILEB;

    // S = Q K^T  (16 x 64 per warp)
    float s[8][4];
#pragma unroll
    for (int j = 0; j < 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int ks2 = 0; ks2 < HD / 32; ++ks2) {
        const int r = j * 8 + (lane & 7);
        const int c = ks2 * 4 + (lane >> 3);
        uint32_t b0, b1, b2, b3;
        ldsm_x4(ks + r * ROWB + ((c ^ (r & 7)) * 16), b0, b1, b2, b3);
        mma_bf16(s[j], qf[2 * ks2], b0, b1);
        mma_bf16(s[j], qf[2 * ks2 + 1], b2, b3);
      }
    }
    // scale, mask, online softmax (rows g and g+8)
    const int key0 = tile * kAttnKeys;
    const bool need_mask = key0 + kAttnKeys > warp_min;
    float tmax[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int j = 0; j < 8; ++j) {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int h = e >> 1;
        float x = s[j][e] * scale2[h];
        if (need_mask) {
          const int key = key0 + j * 8 + 2 * t + (e & 1);
          if (key >= lim[h]) x = -INFINITY;
        }
        s[j][e] = x;
        tmax[h] = fmaxf(tmax[h], x);
      }
    }
    float corr[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      tmax[h] = fmaxf(tmax[h], __shfl_xor_sync(0xffffffffu, tmax[h], 1));
      tmax[h] = fmaxf(tmax[h], __shfl_xor_sync(0xffffffffu, tmax[h], 2));
      const float nm = fmaxf(row_m[h], tmax[h]);
      const float base = nm == -INFINITY ? 0.f : nm;
      corr[h] = exp2f(row_m[h] - base);
      row_m[h] = nm;
      tmax[h] = base;  // reuse as subtraction base
    }
    float tsum[2] = {0.f, 0.f};
    uint32_t pf[4][4];  // P as A fragments for 4 key k-steps
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      float p0 = exp2f(s[j][0] - tmax[0]);
      float p1 = exp2f(s[j][1] - tmax[0]);
      float p2 = exp2f(s[j][2] - tmax[1]);
      float p3 = exp2f(s[j][3] - tmax[1]);
      tsum[0] += p0 + p1;
      tsum[1] += p2 + p3;
      const int kk = j >> 1;
      if ((j & 1) == 0) {
        pf[kk][0] = pack_bf16(p0, p1);
        pf[kk][1] = pack_bf16(p2, p3);
      } else {
        pf[kk][2] = pack_bf16(p0, p1);
        pf[kk][3] = pack_bf16(p2, p3);
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      tsum[h] += __shfl_xor_sync(0xffffffffu, tsum[h], 1);
      tsum[h] += __shfl_xor_sync(0xffffffffu, tsum[h], 2);
      row_l[h] = row_l[h] * corr[h] + tsum[h];
    }
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) {
      o_acc[n][0] *= corr[0];
      o_acc[n][1] *= corr[0];
      o_acc[n][2] *= corr[1];
      o_acc[n][3] *= corr[1];
    }
    // O += P V
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int u = 0; u < HD / 16; ++u) {
        const int r = kk * 16 + ((lane >> 3) & 1) * 8 + (lane & 7);
        const int c = 2 * u + (lane >> 4);
        uint32_t b0, b1, b2, b3;
        ldsm_x4_t(vs + r * ROWB + ((c ^ (r & 7)) * 16), b0, b1, b2, b3);
        mma_bf16(o_acc[2 * u], pf[kk], b0, b1);
        mma_bf16(o_acc[2 * u + 1], pf[kk], b2, b3);
      }
    }
    __syncthreads();
  }
  // normalise and store
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    if (!valid[h]) continue;
    const float inv = row_l[h] > 0.f ? 1.f / row_l[h] : 0.f;
    __nv_bfloat16* o = out + orow_off[h];
#pragma unroll
    for (int n = 0; n < HD / 8; ++n) {
      const int c = n * 8 + 2 * t;
      *reinterpret_cast<__nv_bfloat162*>(o + c) =
          __floats2bfloat162_rn(o_acc[n][2 * h] * inv, o_acc[n][2 * h + 1] * inv);
    }
  }
}

}  // namespace cc

using namespace cc;

extern "C" int cc_sparse_row_attention_mma(const void* q, int64_t ldq, const int64_t* positions, int64_t m,
                                       const void* k_cache, const void* v_cache, int64_t n_keys, int32_t n_q_heads,
                                       int32_t n_kv_heads, int32_t head_dim, float factor, const float* row_factor,
                                       void* out, int64_t ldo, void* stream) {
  CC_CHECK_ARG(n_kv_heads > 0 && n_q_heads % n_kv_heads == 0, CC_ERR_DIMENSION,
               "query heads %d not a multiple of kv heads %d", n_q_heads, n_kv_heads);
  CC_CHECK_ARG(head_dim == 64 || head_dim == 128, CC_ERR_UNSUPPORTED, "head_dim %d unsupported", head_dim);
  CC_CHECK_ARG(n_keys > 0, CC_ERR_VALUE, "attention row with no visible keys");
  if (m <= 0) return CC_OK;
  const int G = n_q_heads / n_kv_heads;
  const int64_t tiles = (m * G + kAttnRows - 1) / kAttnRows;
  dim3 grid((unsigned)tiles, n_kv_heads);
  const int smem = 2 * 2 * kAttnKeys * head_dim * 2;
  cudaStream_t st = as_stream(stream);
  ProfScope ps(st, OP_ATTENTION_MMA, 0);
  if (head_dim == 128) {
    set_smem_once<sparse_row_attention_kernel<128>>(smem);
    sparse_row_attention_kernel<128><<<grid, kAttnThreads, smem, st>>>(
        (const __nv_bfloat16*)q, ldq, positions, m, (const __nv_bfloat16*)k_cache, (const __nv_bfloat16*)v_cache,
        n_keys, n_q_heads, n_kv_heads, factor, row_factor, (__nv_bfloat16*)out, ldo);
  } else {
    sparse_row_attention_kernel<64><<<grid, kAttnThreads, smem, st>>>(
        (const __nv_bfloat16*)q, ldq, positions, m, (const __nv_bfloat16*)k_cache, (const __nv_bfloat16*)v_cache,
        n_keys, n_q_heads, n_kv_heads, factor, row_factor, (__nv_bfloat16*)out, ldo);
  }
  CC_LAUNCH_CHECK("sparse_row_attention");
  return CC_OK;
}
