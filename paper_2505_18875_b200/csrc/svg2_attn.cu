// svg2_attn.cu — A9 (+ fused A10): dynamic-block-size sparse attention over the permuted, cluster-contiguous
// tokens, written for sm_100a.
//
// Work item = two 128-row Q tiles of one query cluster i (contiguous rows of Q' after the permutation) sharing
// ONE packed key stream: the concatenation of the selected key clusters' row ranges of K'/V' (adjacent selected
// clusters merged into runs).  The paper loads K/V "sparsely per token via address offsets into contiguous
// shared memory"; here every 128-key tile of the packed stream is assembled by TMA gather4 (4
// arbitrary rows per instruction) straight into 128B-swizzled shared memory, so there is no per-cluster padding:
// only the last tile of a stream is partial (its N is rounded up to 16 and the tail columns are masked).
//
// Warp roles (384 threads, 1 CTA per SM, persistent over the work list):
//   warp 0      TMA producer: Q tiles (box loads), K/V tiles (gather4) into a 2-stage ring each
//   warp 1      MMA issuer (one thread): S = Q K^T (SS, K-major both) into TMEM; O += P V (TS: P read from TMEM,
//               V MN-major) -- ping-pong order PV_a(t), S_a(t+1), PV_b(t), S_b(t+1)
//   warp 2      TMEM allocator (512 columns: S_a | S_b | O_a | O_b)
//   warps 4-7   softmax warpgroup for Q tile a; warps 8-11 for Q tile b.  One thread = one query row = one TMEM
//               lane: tcgen05.ld S, online softmax in registers (exp2 domain, lazy rescale when the running max
//               grows by > 8), P (bf16) written back over S with tcgen05.st, O rescaled in TMEM when needed;
//               epilogue O / l -> bf16 -> global, scattered to original token order through pi_q (fused A10).
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include "internal.h"
#include "ptx.cuh"
#include "tmap.h"

namespace svg2 {
namespace {

constexpr int kThreads = 384;
constexpr int kStages = 2;
constexpr float kRescaleThreshold = 8.0f;  // log2 units: P <= 256 between rescales
constexpr int kRunSentinelLen = 1 << 20;
// setmaxnreg budget: the launch reserves 168 regs x 384 threads; warpgroup 0 (producer / MMA / TMEM) shrinks to
// 72 and the two softmax warpgroups grow to 216.  The sum must not exceed the reservation or .inc never returns.
constexpr int kRegsCtl = 72, kRegsSoftmax = 216, kRegsLaunch = 168;
static_assert(128 * kRegsCtl + 256 * kRegsSoftmax <= kRegsLaunch * kThreads, "setmaxnreg budget exceeds launch");

template <int D>
struct Cfg {
  static constexpr int kBlocks = D / 64;               // 64-column (128-byte) swizzle blocks per row
  static constexpr uint32_t kBlockBytes = 128 * 128;   // one 64-column block of a 128-row tile
  static constexpr uint32_t kTileBytes = kBlocks * kBlockBytes;
  static constexpr uint32_t kSmemBytes = (2 + 2 * kStages) * kTileBytes + 1024;
  static constexpr uint32_t kColSa = 0, kColSb = 128, kColOa = 256, kColOb = 384;
};

struct Bars {
  uint64_t q_full, q_empty;
  uint64_t k_full[kStages], k_empty[kStages], v_full[kStages], v_empty[kStages];
  uint64_t s_full[2], p_full[2], o_full[2], o_empty[2];
};

struct Params {
  const int4* items;
  const int32_t* n_items;
  const int2* runs;
  const int32_t* run_count;
  const int32_t* nkeys;
  const int32_t* q_perm;
  __nv_bfloat16* O;
  float* lse;
  int Nq, Ck;
  float scale_log2;
};

__device__ __forceinline__ int item_keys(const Params& p, int4 it) { return __ldg(p.nkeys + it.z); }

// The 4 key rows lane `lane` gathers for tile positions [4*lane, 4*lane+4) of the packed stream.
// State (r, off): the tile starts at offset `off` inside run r of this item's run list.  Runs are read 32 at a
// time (one per lane); an inclusive prefix over their lengths resolves each position with a 5-step shuffle
// binary search.  Positions past the end of the stream get the stream's first row (masked later).
__device__ __forceinline__ void tile_rows(const int2* __restrict__ runs, int rc, int& r, int& off, int tile_base,
                                          int nkeys, int lane, int (&rows)[4]) {
  int first_row = __ldg(&runs[0].x);
  bool done[4] = {false, false, false, false};
#pragma unroll
  for (int c = 0; c < 4; ++c) rows[c] = first_row;
  int base = 0;  // tile-relative position where the current window starts
  int wr = r, woff = off;
  while (true) {
    int2 run = (wr + lane < rc) ? __ldg(runs + wr + lane) : make_int2(first_row, kRunSentinelLen);
    int len = run.y - (lane == 0 ? woff : 0);
    int start = run.x + (lane == 0 ? woff : 0);
    int incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const int covered = __shfl_sync(0xffffffffu, incl, 31);
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int P = 4 * lane + c - base;
      // first window lane j with incl_j > P
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int v = __shfl_sync(0xffffffffu, incl, lo + step - 1);
        if (v <= P) lo += step;
      }
      const int ij = __shfl_sync(0xffffffffu, incl, lo);
      const int lj = __shfl_sync(0xffffffffu, len, lo);
      const int sj = __shfl_sync(0xffffffffu, start, lo);
      if (!done[c] && P >= 0 && P < covered) {
        const int gpos = tile_base + 4 * lane + c;
        rows[c] = gpos < nkeys ? sj + (P - (ij - lj)) : first_row;
        done[c] = true;
      }
    }
    if (base + covered >= kKTile) {
      // next tile starts at window position kKTile - base
      const int Pn = kKTile - base;
      int lo = 0;
#pragma unroll
      for (int step = 16; step > 0; step >>= 1) {
        const int v = __shfl_sync(0xffffffffu, incl, lo + step - 1);
        if (v <= Pn) lo += step;
      }
      const int ij = __shfl_sync(0xffffffffu, incl, lo);
      const int lj = __shfl_sync(0xffffffffu, len, lo);
      r = wr + lo;
      off = (lo == 0 ? woff : 0) + (Pn - (ij - lj));
      return;
    }
    base += covered;
    wr += 32;
    woff = 0;
  }
}

template <int D>
__global__ void __launch_bounds__(kThreads, 1)
    k_varblock_attn(const __grid_constant__ CUtensorMap mapQ, const __grid_constant__ CUtensorMap mapK,
                    const __grid_constant__ CUtensorMap mapV, const Params p) {
  using C = Cfg<D>;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = smem;                                // [2][tile]
  uint8_t* sK = smem + 2 * C::kTileBytes;            // [kStages][tile]
  uint8_t* sV = sK + kStages * C::kTileBytes;        // [kStages][tile]
  __shared__ Bars bars;
  __shared__ uint32_t tmem_slot;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&mapQ);
    tma_prefetch_desc(&mapK);
    tma_prefetch_desc(&mapV);
    mbar_init(&bars.q_full, 1);
    mbar_init(&bars.q_empty, 1);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&bars.k_full[s], 1);
      mbar_init(&bars.k_empty[s], 1);
      mbar_init(&bars.v_full[s], 1);
      mbar_init(&bars.v_empty[s], 1);
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&bars.s_full[g], 1);
      mbar_init(&bars.p_full[g], 4);
      mbar_init(&bars.o_full[g], 1);
      mbar_init(&bars.o_empty[g], 4);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<512>(&tmem_slot);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  const int n_items = __ldg(p.n_items);

  if (warp < 4) {
  reg_dealloc<kRegsCtl>();
  if (warp == 0) {
    // ============================ TMA producer ============================
    uint32_t qph = 0, ks = 0, kph = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int4 it = __ldg(p.items + item);
      const int na = it.y & 0xFFFF, nb = it.y >> 16;
      const int nkeys = item_keys(p, it);
      const int2* runs = p.runs + size_t(it.z) * p.Ck;
      const int rc = __ldg(p.run_count + it.z);
      mbar_wait(&bars.q_empty, qph ^ 1, 1);
      if (lane == 0) {
        mbar_arrive_expect_tx(&bars.q_full, (nb > 0 ? 2u : 1u) * C::kTileBytes);
        for (int b = 0; b < C::kBlocks; ++b) {
          tma_load_2d(sQ + b * C::kBlockBytes, &mapQ, &bars.q_full, 64 * b, it.x);
          if (nb > 0) tma_load_2d(sQ + C::kTileBytes + b * C::kBlockBytes, &mapQ, &bars.q_full, 64 * b, it.x + 128);
        }
      }
      qph ^= 1;
      (void)na;
      int r = 0, off = 0;
      const int T = (nkeys + kKTile - 1) / kKTile;
      for (int t = 0; t < T; ++t) {
        int rows[4];
        tile_rows(runs, rc, r, off, t * kKTile, nkeys, lane, rows);
        mbar_wait(&bars.k_empty[ks], kph ^ 1, 2);
        if (lane == 0) mbar_arrive_expect_tx(&bars.k_full[ks], C::kTileBytes);
        __syncwarp();
        uint8_t* dk = sK + ks * C::kTileBytes + lane * 512;
        for (int b = 0; b < C::kBlocks; ++b)
          tma_gather4(dk + b * C::kBlockBytes, &mapK, &bars.k_full[ks], 64 * b, rows[0], rows[1], rows[2], rows[3]);
        mbar_wait(&bars.v_empty[ks], kph ^ 1, 3);
        if (lane == 0) mbar_arrive_expect_tx(&bars.v_full[ks], C::kTileBytes);
        __syncwarp();
        uint8_t* dv = sV + ks * C::kTileBytes + lane * 512;
        for (int b = 0; b < C::kBlocks; ++b)
          tma_gather4(dv + b * C::kBlockBytes, &mapV, &bars.v_full[ks], 64 * b, rows[0], rows[1], rows[2], rows[3]);
        if (++ks == kStages) {
          ks = 0;
          kph ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ============================ MMA issuer ============================
    uint32_t qph = 0, ks = 0, kph = 0, vs = 0, vph = 0;
    uint32_t sph[2] = {0, 0}, oeph[2] = {0, 0};
    (void)sph;
    uint32_t pph[2] = {0, 0};
    const uint32_t idesc_pv = idesc_bf16_f32(128, D, true);
    const uint32_t sQa = smem_u32(sQ), sQb = smem_u32(sQ + C::kTileBytes);
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int4 it = __ldg(p.items + item);
      const bool has_b = (it.y >> 16) > 0;
      const int nkeys = item_keys(p, it);
      const int T = (nkeys + kKTile - 1) / kKTile;
      auto issue_s = [&](int t, int g, uint32_t kstage) {
        const int nvalid = min(kKTile, nkeys - t * kKTile);
        const uint32_t Nt = (uint32_t(nvalid) + 15u) & ~15u;
        const uint32_t idesc = idesc_bf16_f32(128, Nt, false);
        const uint32_t qa = g == 0 ? sQa : sQb;
        const uint32_t kb = smem_u32(sK + kstage * C::kTileBytes);
        const uint32_t dcol = tmem + (g == 0 ? C::kColSa : C::kColSb);
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k >> 2) * C::kBlockBytes + (k & 3) * 32;
          mma_ss(dcol, desc_kmajor_sw128(qa + off), desc_kmajor_sw128(kb + off), idesc, k > 0);
        }
      };
      auto issue_pv = [&](int t, int g, uint32_t vstage) {
        const int nvalid = min(kKTile, nkeys - t * kKTile);
        const int ksteps = (nvalid + 15) / 16;
        const uint32_t vb = smem_u32(sV + vstage * C::kTileBytes);
        const uint32_t pcol = tmem + (g == 0 ? C::kColSa : C::kColSb);
        const uint32_t dcol = tmem + (g == 0 ? C::kColOa : C::kColOb);
        for (int k = 0; k < ksteps; ++k)
          mma_ts(dcol, pcol + 8 * k, desc_mnmajor_sw128(vb + k * 16 * 128, C::kBlockBytes), idesc_pv,
                 (t > 0 || k > 0) ? 1u : 0u);
      };
      mbar_wait(&bars.q_full, qph, 4);
      qph ^= 1;
      // prologue: S(0)
      mbar_wait(&bars.k_full[ks], kph, 5);
      tc_fence_after();
      if (lane == 0) {
        issue_s(0, 0, ks);
        mma_commit(&bars.s_full[0]);
        if (has_b) {
          issue_s(0, 1, ks);
          mma_commit(&bars.s_full[1]);
        }
        mma_commit(&bars.k_empty[ks]);
        if (T == 1) mma_commit(&bars.q_empty);
      }
      __syncwarp();
      if (++ks == kStages) {
        ks = 0;
        kph ^= 1;
      }
      for (int t = 0; t < T; ++t) {
        const bool more = t + 1 < T;
        mbar_wait(&bars.v_full[vs], vph, 6);
        if (more) mbar_wait(&bars.k_full[ks], kph, 7);
        // ---- tile a
        mbar_wait(&bars.p_full[0], pph[0], 8);
        pph[0] ^= 1;
        if (t == 0) {
          mbar_wait(&bars.o_empty[0], oeph[0] ^ 1, 9);
          oeph[0] ^= 1;
        }
        tc_fence_after();
        if (lane == 0) {
          issue_pv(t, 0, vs);
          if (more) {
            issue_s(t + 1, 0, ks);
            mma_commit(&bars.s_full[0]);
          } else {
            mma_commit(&bars.o_full[0]);
          }
        }
        __syncwarp();
        // ---- tile b
        if (has_b) {
          mbar_wait(&bars.p_full[1], pph[1], 10);
          pph[1] ^= 1;
          if (t == 0) {
            mbar_wait(&bars.o_empty[1], oeph[1] ^ 1, 11);
            oeph[1] ^= 1;
          }
          tc_fence_after();
          if (lane == 0) {
            issue_pv(t, 1, vs);
            if (more) {
              issue_s(t + 1, 1, ks);
              mma_commit(&bars.s_full[1]);
            } else {
              mma_commit(&bars.o_full[1]);
            }
          }
          __syncwarp();
        }
        if (lane == 0) {
          mma_commit(&bars.v_empty[vs]);
          if (more) {
            mma_commit(&bars.k_empty[ks]);
            if (t + 2 == T) mma_commit(&bars.q_empty);
          }
        }
        __syncwarp();
        if (++vs == kStages) {
          vs = 0;
          vph ^= 1;
        }
        if (more && ++ks == kStages) {
          ks = 0;
          kph ^= 1;
        }
      }
    }
  }
  } else {
    reg_alloc<kRegsSoftmax>();
    // ============================ softmax warpgroups ============================
    const int g = (warp - 4) >> 2;                  // 0: tile a, 1: tile b
    const int rloc = ((warp & 3) << 5) + lane;      // row in the tile == TMEM lane
    const uint32_t lane_addr = uint32_t((warp & 3) * 32) << 16;
    const uint32_t tS = tmem + lane_addr + (g == 0 ? C::kColSa : C::kColSb);
    const uint32_t tO = tmem + lane_addr + (g == 0 ? C::kColOa : C::kColOb);
    uint32_t sph = 0, oph = 0;
    for (int item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int4 it = __ldg(p.items + item);
      const int nrows = g == 0 ? (it.y & 0xFFFF) : (it.y >> 16);
      if (nrows <= 0) continue;
      const int nkeys = item_keys(p, it);
      const int T = (nkeys + kKTile - 1) / kKTile;
      float m_used = -INFINITY, l = 0.f;
      for (int t = 0; t < T; ++t) {
        const int nvalid = min(kKTile, nkeys - t * kKTile);
        mbar_wait(&bars.s_full[g], sph, 12 + g);
        sph ^= 1;
        tc_fence_after();
        uint32_t s0[32], s1[32], s2[32], s3[32];
        tmem_ld32(tS + 0, s0);
        tmem_ld32(tS + 32, s1);
        tmem_ld32(tS + 64, s2);
        tmem_ld32(tS + 96, s3);
        tmem_wait_ld();
        float mt = -INFINITY;
        const float sl2 = p.scale_log2;
        auto scale_mask = [&](uint32_t(&a)[32], int c0) {
#pragma unroll
          for (int e = 0; e < 32; ++e) {
            const float x = (c0 + e < nvalid) ? __uint_as_float(a[e]) * sl2 : -INFINITY;
            a[e] = __float_as_uint(x);
            mt = fmaxf(mt, x);
          }
        };
        scale_mask(s0, 0);
        scale_mask(s1, 32);
        scale_mask(s2, 64);
        scale_mask(s3, 96);
        if (t == 0) {
          m_used = mt;
        } else if (__any_sync(0xffffffffu, mt > m_used + kRescaleThreshold)) {
          // warp-uniform branch (tcgen05.ld/st are .sync.aligned); rows whose max did not grow get alpha = 1
          const float m_new = fmaxf(m_used, mt);
          const float alpha = ex2_approx(m_used - m_new);
          l *= alpha;
#pragma unroll 1
          for (int c = 0; c < D / 32; ++c) {
            uint32_t o[32];
            tmem_ld32(tO + 32 * c, o);
            tmem_wait_ld();
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = __float_as_uint(__uint_as_float(o[e]) * alpha);
            tmem_st32(tO + 32 * c, o);
          }
          m_used = m_new;
        }
        float lsum = 0.f;
        auto exp_store = [&](const uint32_t(&a)[32], int c) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) {
            const float p0 = ex2_approx(__uint_as_float(a[2 * e]) - m_used);
            const float p1 = ex2_approx(__uint_as_float(a[2 * e + 1]) - m_used);
            lsum += p0 + p1;
            pk[e] = pack_bf16x2(p0, p1);
          }
          tmem_st16(tS + 16 * c, pk);
        };
        exp_store(s0, 0);
        exp_store(s1, 1);
        exp_store(s2, 2);
        exp_store(s3, 3);
        l += lsum;
        tmem_wait_st();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&bars.p_full[g]);
      }
      // ---- epilogue: O / l  -> bf16 -> original token order (fused pi_q^T)
      mbar_wait(&bars.o_full[g], oph, 14 + g);
      oph ^= 1;
      tc_fence_after();
      const float inv_l = 1.f / l;
      const long long row_flat = (long long)it.x + g * kQTile + rloc;
      long long dst = row_flat;
      if (rloc < nrows && p.q_perm) {
        const long long bh = it.w;
        dst = bh * p.Nq + __ldg(p.q_perm + row_flat);
      }
      uint4* orow = reinterpret_cast<uint4*>(p.O + dst * D);
#pragma unroll
      for (int c = 0; c < D / 32; ++c) {
        uint32_t o[32];
        tmem_ld32(tO + 32 * c, o);
        tmem_wait_ld();
        if (rloc < nrows) {
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            uint4 u;
            u.x = pack_bf16x2(__uint_as_float(o[8 * v + 0]) * inv_l, __uint_as_float(o[8 * v + 1]) * inv_l);
            u.y = pack_bf16x2(__uint_as_float(o[8 * v + 2]) * inv_l, __uint_as_float(o[8 * v + 3]) * inv_l);
            u.z = pack_bf16x2(__uint_as_float(o[8 * v + 4]) * inv_l, __uint_as_float(o[8 * v + 5]) * inv_l);
            u.w = pack_bf16x2(__uint_as_float(o[8 * v + 6]) * inv_l, __uint_as_float(o[8 * v + 7]) * inv_l);
            orow[4 * c + v] = u;
          }
        }
      }
      if (rloc < nrows && p.lse) p.lse[dst] = (m_used + __log2f(l)) * 0.69314718055994531f;
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&bars.o_empty[g]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------------- work-list builder
constexpr int kBuildThreads = 256;

// per (b,h): runs of selected, non-empty key clusters (ascending j, contiguous ones merged), key counts, and
// the work items (pairs of 128-row Q tiles) of every non-empty query cluster, in (i, tile) order.
__global__ void __launch_bounds__(kBuildThreads) k_build(const int32_t* __restrict__ q_off, const int32_t* __restrict__ k_off,
                                                         const uint8_t* __restrict__ mask, int Nq, int Nk, int Cq,
                                                         int Ck, int cap, AttnWs ws) {
  const int bh = blockIdx.x, tid = threadIdx.x;
  const int per = (Cq + kBuildThreads - 1) / kBuildThreads;
  const int i0 = min(Cq, tid * per), i1 = min(Cq, i0 + per);
  const int32_t* qo = q_off + size_t(bh) * (Cq + 1);
  const int32_t* ko = k_off + size_t(bh) * (Ck + 1);
  int my_items = 0;
  for (int i = i0; i < i1; ++i) {
    const size_t li = size_t(bh) * Cq + i;
    const uint8_t* mrow = mask + li * Ck;
    int2* runs = ws.runs + li * Ck;
    int cnt = 0, keys = 0, cs = -1, ce = -1;
    for (int j = 0; j < Ck; ++j) {
      if (!mrow[j]) continue;
      const int s = __ldg(ko + j), e = __ldg(ko + j + 1);
      if (e <= s) continue;
      if (s == ce) {
        ce = e;
      } else {
        if (cs >= 0) {
          runs[cnt++] = make_int2(int(size_t(bh) * Nk) + cs, ce - cs);
          keys += ce - cs;
        }
        cs = s;
        ce = e;
      }
    }
    if (cs >= 0) {
      runs[cnt++] = make_int2(int(size_t(bh) * Nk) + cs, ce - cs);
      keys += ce - cs;
    }
    ws.run_count[li] = cnt;
    ws.nkeys[li] = keys;
    const int sq = __ldg(qo + i + 1) - __ldg(qo + i);
    if (keys > 0) my_items += (sq + kItemRows - 1) / kItemRows;
  }
  // exclusive scan of my_items across the block
  __shared__ int warp_tot[kBuildThreads / 32];
  int x = my_items;
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, o);
    if ((tid & 31) >= o) x += y;
  }
  if ((tid & 31) == 31) warp_tot[tid >> 5] = x;
  __syncthreads();
  int before = 0, total = 0;
  for (int w = 0; w < kBuildThreads / 32; ++w) {
    if (w < (tid >> 5)) before += warp_tot[w];
    total += warp_tot[w];
  }
  int slot = before + x - my_items;
  int4* out = ws.items_bh + size_t(bh) * cap;
  for (int i = i0; i < i1; ++i) {
    const size_t li = size_t(bh) * Cq + i;
    const int q0 = __ldg(qo + i), sq = __ldg(qo + i + 1) - q0;
    if (ws.nkeys[li] <= 0) continue;
    for (int u = 0; u * kItemRows < sq; ++u) {
      const int rem = sq - u * kItemRows;
      const int na = min(kQTile, rem), nb = max(0, min(kQTile, rem - kQTile));
      out[slot++] = make_int4(int(size_t(bh) * Nq) + q0 + u * kItemRows, na | (nb << 16), int(li), bh);
    }
  }
  if (tid == 0) ws.items_cnt[bh] = total;
}

__global__ void __launch_bounds__(1024) k_flatten(int BH, int cap, AttnWs ws) {
  int base = 0;
  for (int bh = 0; bh < BH; ++bh) {
    const int cnt = ws.items_cnt[bh];
    for (int t = threadIdx.x; t < cnt; t += blockDim.x) ws.items[base + t] = ws.items_bh[size_t(bh) * cap + t];
    base += cnt;
  }
  if (threadIdx.x == 0) *ws.n_items = base;
}

template <int D>
cudaError_t run_attn(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, int Ck, float scale,
                     const int32_t* q_perm, void* O, float* lse, AttnWs ws, cudaStream_t s) {
  CUtensorMap mq, mk, mv;
  if (!make_tmap_bf16(&mq, Qp, uint64_t(BH) * Nq, D, 128) || !make_tmap_bf16(&mk, Kp, uint64_t(BH) * Nk, D, 1) ||
      !make_tmap_bf16(&mv, Vp, uint64_t(BH) * Nk, D, 1))
    return cudaErrorInvalidValue;
  Params p;
  p.items = ws.items;
  p.n_items = ws.n_items;
  p.runs = ws.runs;
  p.run_count = ws.run_count;
  p.nkeys = ws.nkeys;
  p.q_perm = q_perm;
  p.O = static_cast<__nv_bfloat16*>(O);
  p.lse = lse;
  p.Nq = Nq;
  p.Ck = Ck;
  p.scale_log2 = scale * 1.4426950408889634f;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaFuncSetAttribute(k_varblock_attn<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg<D>::kSmemBytes);
  k_varblock_attn<D><<<sms, kThreads, Cfg<D>::kSmemBytes, s>>>(mq, mk, mv, p);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_build_worklist(const int32_t* q_offsets, const int32_t* k_offsets, const uint8_t* mask, int BH,
                                  int Nq, int Nk, int Cq, int Ck, AttnWs ws, cudaStream_t s) {
  const int cap = items_cap_per_bh(Nq, Cq);
  k_build<<<BH, kBuildThreads, 0, s>>>(q_offsets, k_offsets, mask, Nq, Nk, Cq, Ck, cap, ws);
  k_flatten<<<1, 1024, 0, s>>>(BH, cap, ws);
  return cudaGetLastError();
}

cudaError_t launch_varblock_attention(const void* Qp, const void* Kp, const void* Vp, int BH, int Nq, int Nk, int d,
                                      int Cq, int Ck, float scale, const int32_t* q_perm, void* O, float* lse,
                                      AttnWs ws, cudaStream_t s) {
  (void)Cq;
  if (d == 128) return run_attn<128>(Qp, Kp, Vp, BH, Nq, Nk, Ck, scale, q_perm, O, lse, ws, s);
  return run_attn<64>(Qp, Kp, Vp, BH, Nq, Nk, Ck, scale, q_perm, O, lse, ws, s);
}

}  // namespace svg2
