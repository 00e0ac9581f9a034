// Hessian assembly on the FP64 tensor pipe (DMMA).
//
// -H = sum_i J_i^T (diag p_i - p_i p_i^T) J_i is split into three contractions over the
// individuals i, each a sum of rank-1 terms whose factors are generated on chip from the
// per-individual rows Pr = [P_i | ybar_i], Xp = [1 | x_i], Zp = [z_i] (never an N x n_p matrix):
//
//  J1  beta-beta (Eq. "hessian block" case 1 with M = X):
//        -H[(k,a),(l,b)] = sum_i w_kl,i x~_ia x~_ib,  w_kl,i = P_ik (delta_kl - P_il)
//      computed for k <= l (block symmetry P:484) AND a <= b (each block is symmetric since
//      x~ x~^T is): one GEMM  C1[pair(k,l)][vech(a,b)] = sum_i W[i][pair] * S[i][vech],
//      W[i][(k,l)] = P_ik (delta_kl - P_il) and S[i][(a,b)] = x~_ia x~_ib generated in smem —
//      each X tile is staged once and reused for every (k,l) weight pair of the output tile.
//  J2  blocks touching the alternative-specific Z or the generic Y (cases 1-3 of P:469-471 with
//      M = Z_k, and the O(K) regrouping of the generic blocks):
//        U[i][r] = sum_k P_ik J_i[k][r]  (= P_ik m_ik for beta/alpha columns, ybar_i for gamma)
//        C2 = U^T U restricted to columns alpha u gamma  (rows: all n_p)
//  J3  the same-alternative ("delta_kl") terms of those blocks, per alternative k:
//        T_k = sum_i P_ik e_ik f_ik^T,  e = [x~_i, z_ik, y_ik], f = [z_ik, y_ik]
//  so that  -H = C1 (beta-beta)  and  -H = T - C2 (every other entry).
//
// J1/J2 run warp-level DMMA kernels (mma.sync.m8n8k4.f64 — tcgen05 has no f64 kind on sm_100a)
// over 128 x BN output tiles, inner dimension = individuals in chunks of KC. Default: both operands
// are materialised per chunk in fragment-native order by k_frag (W every evaluation, the design
// products once per design; J2's A and B in one pass) and k_pipe_gemm streams them with one
// cp.async.bulk each into an mbarrier ring (1 producer warp, 8 consumer warps issuing DMMAs only).
// Fallback (k_gen_gemm): the raw rows are fetched by cp.async.bulk into a stage and every thread
// generates its fragment-native operand elements (v = R[o1] * (c0 + s R[o2])) on chip.
// Split-N partial tiles are reduced in a fixed order (deterministic), then k_assemble gathers
// H (exactly symmetric) into the caller's row-major n_p x n_p buffer.
#include <algorithm>
#include <cstdlib>
#include <cstdio>
#include <vector>

#include "internal.h"

namespace mnl {

struct ColDesc {
  int o1, ld1, o2, ld2;  // stage offsets (doubles) of the two factors for row 0, and row strides
  double c0, s;          // value = R[o1] * (c0 + s * R[o2])
};

namespace {

constexpr int BM = 128;

struct GemmParams {
  const ColDesc* descA;
  const ColDesc* descB;
  int tilesM, tilesN, splits;
  int64_t nchunks;
  int64_t cstride;  // chunk dimension of the fragment buffers (k_pipe_gemm; = nchunks unless N-slabbed)
  double* C;
  int ldc;
  int64_t split_stride;
  int nseg;
  const double* seg_ptr[3];
  int seg_ld[3];
  int seg_off[3];
  int stage_doubles;
  unsigned stage_bytes;
  int nraw;  // raw stages: 2 (prefetch two chunks ahead) or 1 (refill after the generate phase)
  const double* bfrag;  // BPRE: B operand precomputed in fragment-native order [tilesN][nchunks][GB_D]
  unsigned* counter;
  // >= 0: skip the tiles whose every row r exceeds skip_off + every column c (J2: the lower
  // triangle of the symmetric Z/Y x Z/Y block, never read by the assembly, which takes (min, max))
  int skip_off;
};
__host__ __device__ __forceinline__ bool skip_tile(int skip_off, int tm, int tn, int bn) {
  return skip_off >= 0 && (int64_t)tm * 128 > (int64_t)skip_off + (int64_t)tn * bn + bn - 1;
}

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_stage(const GemmParams& P, double* dst, int64_t chunk, int KC,
                                          uint64_t* bar) {
  const unsigned b = smem_u32(bar);
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(P.stage_bytes)
               : "memory");
  for (int s = 0; s < P.nseg; ++s) {
    const double* src = P.seg_ptr[s] + chunk * KC * (int64_t)P.seg_ld[s];
    const unsigned bytes = (unsigned)(KC * P.seg_ld[s] * 8);
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst + P.seg_off[s])),
        "l"(src), "r"(bytes), "r"(b)
        : "memory");
  }
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  // volatile: keeps the program order (fragment loads for ks+1 ahead of ks's DMMAs)
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 lds128(const double* p) {
  double2 v;
  asm volatile("ld.shared.v2.f64 {%0,%1}, [%2];" : "=d"(v.x), "=d"(v.y) : "r"(smem_u32(p)));
  return v;
}

struct Gen {  // one generated column, pre-offset to this lane's row (i % 4)
  int p1, s1, p2, s2;
  double c0, s;
};
__device__ __forceinline__ Gen make_gen(const ColDesc& d, int r4) {
  Gen g;
  g.p1 = d.o1 + r4 * d.ld1;
  g.s1 = 4 * d.ld1;
  g.p2 = d.o2 + r4 * d.ld2;
  g.s2 = 4 * d.ld2;
  g.c0 = d.c0;
  g.s = d.s;
  return g;
}

// AGEN: A columns use the general form R1 * (c0 + s R2) (J1's weights P_k (delta_kl - P_l));
// otherwise, and always for B, the descriptors are plain products R1 * R2 (c0 = 0, s = 1).
// BPRE: the B operand does not depend on the probabilities (J1's vech x~ x~^T), so it is precomputed
// once per design in fragment-native order and fetched per chunk by one bulk copy (no generation).
template <int BN, int KC, int NWARP, bool AGEN, bool BPRE = false>
__global__ void __launch_bounds__(NWARP * 32, (NWARP < 8 ? 8 / NWARP : 1)) k_gen_gemm(const GemmParams P) {
  // 8 warps: 128 -> 2x4 warps of 64x32; 96 -> 4x2 of 32x48; 64 -> 4x2 of 32x32.
  // 4 warps (two CTAs per SM): 64 -> 2x2 of 64x32.  16 warps: 128 -> 4x4 of 32x32.
  constexpr int WARPS_M = NWARP == 4 ? 2 : (NWARP == 16 ? 4 : ((BN == 128) ? 2 : 4));
  constexpr int WARPS_N = NWARP / WARPS_M;
  constexpr int WTM = BM / WARPS_M, WTN = BN / WARPS_N;
  constexpr int MT = WTM / 8, NTL = WTN / 8;
  constexpr int KS = KC / 4;
  constexpr int PBA = BM / 16, PBB = BN / 16;
  constexpr int GA_D = KS * PBA * 64, GB_D = KS * PBB * 64;  // doubles per buffer
  // generator work split: warp w handles pair-blocks of group wg (PA_W of A, PB_W of B) for the
  // k-slices of half kh (16 warps: two warps share a pair-block, one k-half each)
  constexpr int KSPLIT = NWARP > 8 ? NWARP / 8 : 1;
  constexpr int NWG = NWARP / KSPLIT;                 // warps per k-slice group
  constexpr int KSW = KS / KSPLIT;                    // k-slices per warp
  constexpr int PA_W = PBA / NWG;                     // A pair-blocks generated per warp
  constexpr int PB_W = (PBB + NWG - 1) / NWG;         // B pair-blocks generated per warp
  static_assert(PBA % NWG == 0, "A pair-blocks must split evenly over the warps");

  extern __shared__ __align__(128) double sm[];
  double* GA = sm;                          // [2][KS][PBA][32][2]
  double* GB = GA + 2 * GA_D;               // [2][KS][PBB][32][2]
  double* RAW = GB + 2 * GB_D;              // [2][stage_doubles]
  __shared__ __align__(8) uint64_t mbar[2];
  __shared__ __align__(8) uint64_t bfull[2];
  __shared__ int s_item;

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  const int wm = w / WARPS_N, wn = w % WARPS_N;
  const int r4 = lane & 3, cl = lane >> 2;
  const int wg = w % NWG, kh = w / NWG;
  auto b_copy = [&](int tn_, int64_t c_, unsigned buf) {  // BPRE: fetch chunk c_'s B fragments
    const unsigned bar = smem_u32(&bfull[buf]);
    constexpr unsigned bytes = GB_D * 8;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
    const double* src = P.bfrag + ((int64_t)tn_ * P.nchunks + c_) * GB_D;
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(GB + buf * GB_D)), "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
  };

  if (tid == 0) {
    mbar_init(&mbar[0], 1);
    mbar_init(&mbar[1], 1);
    mbar_init(&bfull[0], 1);
    mbar_init(&bfull[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  const int tiles = P.tilesM * P.tilesN;
  const int total = tiles * P.splits;
  unsigned gc = 0;  // chunks consumed by this CTA (buffer = gc & 1, parity = (gc >> 1) & 1)

  for (;;) {
    if (tid == 0) s_item = (int)atomicAdd(P.counter, 1u);
    __syncthreads();
    const int item = s_item;
    if (item >= total) break;
    const int split = item / tiles, t = item - split * tiles;
    const int tm = t / P.tilesN, tn = t - tm * P.tilesN;
    if (skip_tile(P.skip_off, tm, tn, BN)) {
      __syncthreads();  // every thread has read s_item before thread 0 fetches the next item
      continue;
    }
    const int64_t c_begin = split * P.nchunks / P.splits;
    const int64_t c_end = (split + 1) * P.nchunks / P.splits;

    // per-thread generator columns (constant over the item): warp w generates A pair-blocks
    // w*PA_W .. and B pair-blocks w*PB_W .. (those < PBB), all ks
    Gen gA[PA_W][2], gBv[PB_W][2];
#pragma unroll
    for (int j = 0; j < PA_W; ++j) {
      const int pb = wg * PA_W + j;
      gA[j][0] = make_gen(P.descA[tm * BM + (2 * pb) * 8 + cl], r4);
      gA[j][1] = make_gen(P.descA[tm * BM + (2 * pb + 1) * 8 + cl], r4);
    }
#pragma unroll
    for (int j = 0; j < PB_W; ++j) {
      const int pb = min(wg * PB_W + j, PBB - 1);
      gBv[j][0] = make_gen(P.descB[tn * BN + (2 * pb) * 8 + cl], r4);
      gBv[j][1] = make_gen(P.descB[tn * BN + (2 * pb + 1) * 8 + cl], r4);
    }

    if (tid == 0) {
      for (int64_t c = c_begin; c < c_end && c < c_begin + P.nraw; ++c) {
        const unsigned b = P.nraw == 2 ? ((gc + (unsigned)(c - c_begin)) & 1u) : 0u;
        tma_stage(P, RAW + b * P.stage_doubles, c, KC, &mbar[b]);
      }
      if constexpr (BPRE) b_copy(tn, c_begin, gc & 1u);
    }

    double acc[MT][NTL][2];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NTL; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

    for (int64_t c = c_begin; c < c_end; ++c, ++gc) {
      const unsigned b = gc & 1u;
      const unsigned rb = P.nraw == 2 ? b : 0u;
      mbar_wait(&mbar[rb], P.nraw == 2 ? ((gc >> 1) & 1u) : (gc & 1u));
      if constexpr (BPRE) mbar_wait(&bfull[b], (gc >> 1) & 1u);
      const double* R = RAW + rb * P.stage_doubles;
      double* ga = GA + b * GA_D;
      double* gb = GB + b * GB_D;
      // ---- generate operand fragments (fragment-native layout, one double2 per lane) ----
      // in batches of GB k-slices: all shared-memory loads of a batch first, then the FP64 ops,
      // then the stores (the accumulators leave ~60 registers free here; latency ~ 1 round trip)
      constexpr int GBT = KSW < 8 ? KSW : 8;
      const int ks0 = kh * KSW;
#pragma unroll
      for (int j = 0; j < PA_W; ++j)
#pragma unroll
        for (int kb = ks0; kb < ks0 + KSW; kb += GBT) {
          double a1[GBT][2], a2[GBT][2];
#pragma unroll
          for (int t = 0; t < GBT; ++t)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              a1[t][h] = R[gA[j][h].p1 + (kb + t) * gA[j][h].s1];
              a2[t][h] = R[gA[j][h].p2 + (kb + t) * gA[j][h].s2];
            }
#pragma unroll
          for (int t = 0; t < GBT; ++t) {
            double2 v;
            if constexpr (AGEN) {
              v.x = a1[t][0] * fma(gA[j][0].s, a2[t][0], gA[j][0].c0);
              v.y = a1[t][1] * fma(gA[j][1].s, a2[t][1], gA[j][1].c0);
            } else {
              v.x = a1[t][0] * a2[t][0];
              v.y = a1[t][1] * a2[t][1];
            }
            reinterpret_cast<double2*>(ga)[((kb + t) * PBA + wg * PA_W + j) * 32 + lane] = v;
          }
        }
#pragma unroll
      for (int j = 0; j < (BPRE ? 0 : PB_W); ++j) {
        const int pb = wg * PB_W + j;
        if (pb < PBB) {
#pragma unroll
          for (int kb = ks0; kb < ks0 + KSW; kb += GBT) {
            double b1[GBT][2], b2[GBT][2];
#pragma unroll
            for (int t = 0; t < GBT; ++t)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                b1[t][h] = R[gBv[j][h].p1 + (kb + t) * gBv[j][h].s1];
                b2[t][h] = R[gBv[j][h].p2 + (kb + t) * gBv[j][h].s2];
              }
#pragma unroll
            for (int t = 0; t < GBT; ++t) {
              double2 v;
              v.x = b1[t][0] * b2[t][0];
              v.y = b1[t][1] * b2[t][1];
              reinterpret_cast<double2*>(gb)[((kb + t) * PBB + pb) * 32 + lane] = v;
            }
          }
        }
      }
      __syncthreads();
      if (tid == 0 && c + P.nraw < c_end) tma_stage(P, RAW + rb * P.stage_doubles, c + P.nraw, KC, &mbar[rb]);
      if constexpr (BPRE)
        if (tid == 0 && c + 1 < c_end) b_copy(tn, c + 1, b ^ 1u);  // its buffer was freed by DMMA(c-1)
      // ---- DMMA on this chunk (fragments for ks+1 loaded while ks's DMMAs issue) ----
      double af[2][MT], bf[2][NTL];
      auto load_frags = [&](int buf, int ks) {
#pragma unroll
        for (int mp = 0; mp < MT / 2; ++mp) {
          const double2 v = lds128(ga + 2 * ((ks * PBA + wm * (MT / 2) + mp) * 32 + lane));
          af[buf][2 * mp] = v.x;
          af[buf][2 * mp + 1] = v.y;
        }
#pragma unroll
        for (int np = 0; np < NTL / 2; ++np) {
          const double2 v = lds128(gb + 2 * ((ks * PBB + wn * (NTL / 2) + np) * 32 + lane));
          bf[buf][2 * np] = v.x;
          bf[buf][2 * np + 1] = v.y;
        }
      };
      load_frags(0, 0);
#pragma unroll
      for (int ks = 0; ks < KS; ++ks) {
        if (ks + 1 < KS) load_frags((ks + 1) & 1, ks + 1);
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < NTL; ++j) dmma(acc[i][j][0], acc[i][j][1], af[ks & 1][i], bf[ks & 1][j]);
      }
    }
    // ---- epilogue: this split's partial tile ----
    double* Cb = P.C + split * P.split_stride;
#pragma unroll
    for (int i = 0; i < MT; ++i) {
      const int64_t row = (int64_t)tm * BM + wm * WTM + i * 8 + cl;
#pragma unroll
      for (int j = 0; j < NTL; ++j) {
        const int col = tn * BN + wn * WTN + j * 8 + 2 * r4;
        *reinterpret_cast<double2*>(Cb + row * P.ldc + col) = make_double2(acc[i][j][0], acc[i][j][1]);
      }
    }
  }
}

// Operand materialisation: the generated columns of one GEMM operand written once to HBM in the
// GEMM kernels' fragment-native order, one CTA per chunk of KC individuals (the chunk's rows of the
// descriptor segments staged once in shared memory, then every tile of the operand written with
// 16-byte coalesced stores). Same arithmetic as the in-kernel generator (k_gen_gemm):
// out[(t * nchunks + c) * GD + ((ks * PB + pb) * 32 + lane) * 2 + h] = R[o1] * fma(s, R[o2], c0) of
//   column t * BT + (2 pb + h) * 8 + lane / 4 at individual c * KC + 4 ks + lane % 4   (GD = KS * PB * 64).
struct FragArgs {
  const ColDesc* desc;
  double* out;
  int tiles, BT, KC;
  int64_t nchunks;  // chunk dimension of the output buffers (the grid covers count <= nchunks chunks)
  int64_t c_base;   // first individual chunk of this launch (N-slab)
  int nseg;
  const double* seg_ptr[3];
  int seg_ld[3];
  int seg_off[3];
  int nh;  // CTAs per chunk (frag_nh: KC / nh staged rows)
  // optional second / third operands from the same staged rows (J2: A, B and the tail's B in one
  // pass); tiles2 / tiles3 = 0: none
  const ColDesc* desc2;
  double* out2;
  int tiles2, BT2;
  const ColDesc* desc3;
  double* out3;
  int tiles3, BT3;
};

// offset into a KC-row stage -> offset into the KC/2-row stage (segment bases halve; the in-row
// column offset stays)
__device__ __forceinline__ int rebase(const FragArgs& F, int o) {
  int sg = 0;
#pragma unroll
  for (int t = 1; t < 3; ++t)
    if (t < F.nseg && o >= F.seg_off[t]) sg = t;
  const int base = sg == 0 ? F.seg_off[0] : (sg == 1 ? F.seg_off[1] : F.seg_off[2]);
  return base / F.nh + (o - base);
}

__global__ void __launch_bounds__(256) k_frag(const FragArgs F) {
  // CTA = (chunk c, part h < nh): rows c * KC + h * KC / nh + [0, KC / nh), k-slices [h KS/nh, (h+1) KS/nh)
  extern __shared__ __align__(16) double rs[];
  const int64_t c = blockIdx.x / F.nh;
  const int h = blockIdx.x - (int)c * F.nh, RH = F.KC / F.nh;
#pragma unroll
  for (int sg = 0; sg < 3; ++sg) {
    if (sg >= F.nseg) break;
    const int n2 = RH * F.seg_ld[sg] / 2;  // leading dimensions are even
    const double2* src =
        reinterpret_cast<const double2*>(F.seg_ptr[sg] + ((F.c_base + c) * F.KC + h * RH) * (int64_t)F.seg_ld[sg]);
    double2* dst = reinterpret_cast<double2*>(rs + F.seg_off[sg] / F.nh);  // seg_off: offsets for KC rows
    for (int e = threadIdx.x; e < n2; e += blockDim.x) dst[e] = src[e];
  }
  __syncthreads();
  // one thread per (tile, pair-block, lane): its two columns' descriptors stay in registers over
  // the k-slices; for each k-slice a warp stores 512 contiguous bytes. Descriptor offsets assume
  // KC staged rows per segment (seg_off = KC * preceding lds): rebase to the half-size stage.
  const int KS = F.KC / 4;
  const int W1 = (F.BT / 16) * 32, W2 = (F.BT2 / 16) * 32, W3 = (F.BT3 / 16) * 32;
  const int n1 = F.tiles * W1, n2 = n1 + F.tiles2 * W2;
  for (int wi = threadIdx.x; wi < n2 + F.tiles3 * W3; wi += blockDim.x) {
    const int which = wi < n1 ? 0 : (wi < n2 ? 1 : 2);  // picks the operand only
    const int w = which == 0 ? wi : (which == 1 ? wi - n1 : wi - n2);
    const int W = which == 0 ? W1 : (which == 1 ? W2 : W3), BT = which == 0 ? F.BT : (which == 1 ? F.BT2 : F.BT3);
    const ColDesc* desc = which == 0 ? F.desc : (which == 1 ? F.desc2 : F.desc3);
    double* outp = which == 0 ? F.out : (which == 1 ? F.out2 : F.out3);
    const int t = w / W, r = w - t * W, lane = r & 31;
    const int col = t * BT + (r >> 5) * 16 + (lane >> 2);
    ColDesc d0 = desc[col], d1 = desc[col + 8];
    d0.o1 = rebase(F, d0.o1); d0.o2 = rebase(F, d0.o2);
    d1.o1 = rebase(F, d1.o1); d1.o2 = rebase(F, d1.o2);
    const int i0 = lane & 3;
    double2* dst = reinterpret_cast<double2*>(outp + ((int64_t)t * F.nchunks + c) * (KS * W * 2)) + r;
#pragma unroll 4
    for (int kq = 0; kq < KS / F.nh; ++kq) {
      const int i = 4 * kq + i0, ks = h * (KS / F.nh) + kq;
      double2 o;
      o.x = rs[d0.o1 + i * d0.ld1] * fma(d0.s, rs[d0.o2 + i * d0.ld2], d0.c0);
      o.y = rs[d1.o1 + i * d1.ld1] * fma(d1.s, rs[d1.o2 + i * d1.ld2], d1.c0);
      __stcs(dst + ks * W, o);  // streamed: the GEMM reads it back from HBM
    }
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Pipelined DMMA GEMM over precomputed fragment-native operands (J1 when both A and B are
// materialised): warp NWARP is the producer (one lane: dynamic item fetch, then per chunk one
// 32 KB bulk copy of A and of B into an S-stage ring guarded by full/empty mbarriers); warps
// 0..NWARP-1 only load fragments and issue DMMA. No CTA-wide barrier inside the loop: a stage is
// refilled as soon as the NWARP consumer warps have released it. Item metadata travels with the
// stage (written before the producer's release-arrive, read after the consumers' acquire-wait).
template <int BN, int KC, int S, int BMT = BM>
__global__ void __launch_bounds__(8 * 32 + 32, 1) k_pipe_gemm(const GemmParams P, const double* __restrict__ afrag) {
  // BMT = 128: 128 -> 2x4 warps of 64x32; 112 -> 8x1 of 16x112; 96 -> 4x2 of 32x48; 64 -> 4x2 of 32x32;
  // 48 -> 8x1 of 16x48. BMT = 64 (few weight pairs): 128 -> 2x4 of 32x32; 96 -> 4x2 of 16x48;
  // 64 -> 2x4 of 32x16.
  constexpr int NWARP = 8;
  constexpr int WARPS_M = BMT == 64 ? (BN == 96 ? 4 : 2)
                                    : ((BN == 128) ? 2 : ((BN == 48 || BN == 112) ? 8 : 4)),
                WARPS_N = NWARP / WARPS_M;
  constexpr int WTM = BMT / WARPS_M, WTN = BN / WARPS_N;
  constexpr int MT = WTM / 8, NTL = WTN / 8;
  constexpr int KS = KC / 4, PBA = BMT / 16, PBB = BN / 16;
  constexpr int GA_D = KS * PBA * 64, GB_D = KS * PBB * 64;
  extern __shared__ __align__(128) double sm[];  // [S][GA_D + GB_D]
  __shared__ __align__(8) uint64_t full[S], empty[S];
  __shared__ int meta_item[S], meta_flags[S];

  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int tiles = P.tilesM * P.tilesN, total = tiles * P.splits;

  if (w == NWARP) {  // producer
    if (lane != 0) return;
    unsigned s = 0, ph = 0;
    for (;;) {
      const int item = (int)atomicAdd(P.counter, 1u);
      if (item >= total) {
        mbar_wait(&empty[s], ph ^ 1u);
        meta_item[s] = -1;
        mbar_arrive(&full[s]);
        return;
      }
      const int split = item / tiles, t = item - split * tiles;
      const int tm = t / P.tilesN, tn = t - tm * P.tilesN;
      if (skip_tile(P.skip_off, tm, tn, BN)) continue;  // never staged: the consumers never see it
      const int64_t cb = split * P.nchunks / P.splits, ce = (split + 1) * P.nchunks / P.splits;
      for (int64_t c = cb; c < ce; ++c) {
        mbar_wait(&empty[s], ph ^ 1u);
        meta_item[s] = item;
        meta_flags[s] = (c == cb ? 1 : 0) | (c + 1 == ce ? 2 : 0);
        double* st = sm + s * (GA_D + GB_D);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                     "r"((unsigned)((GA_D + GB_D) * 8))
                     : "memory");
        bulk_g2s(st, afrag + ((int64_t)tm * P.cstride + c) * GA_D, GA_D * 8, &full[s]);
        bulk_g2s(st + GA_D, P.bfrag + ((int64_t)tn * P.cstride + c) * GB_D, GB_D * 8, &full[s]);
        if (++s == S) { s = 0; ph ^= 1u; }
      }
    }
  }

  // consumers
  const int wm = w / WARPS_N, wn = w % WARPS_N;
  const int r4 = lane & 3, cl = lane >> 2;
  double acc[MT][NTL][2];
  unsigned s = 0, ph = 0;
  for (;;) {
    mbar_wait(&full[s], ph);
    const int item = meta_item[s], fl = meta_flags[s];
    if (item < 0) break;
    if (fl & 1) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTL; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
    }
    const double* ga = sm + s * (GA_D + GB_D);
    const double* gb = ga + GA_D;
    double af[2][MT], bf[2][NTL];
    auto load_frags = [&](int buf, int ks) {
#pragma unroll
      for (int mp = 0; mp < MT / 2; ++mp) {
        const double2 v = lds128(ga + 2 * ((ks * PBA + wm * (MT / 2) + mp) * 32 + lane));
        af[buf][2 * mp] = v.x;
        af[buf][2 * mp + 1] = v.y;
      }
#pragma unroll
      for (int np = 0; np < NTL / 2; ++np) {
        const double2 v = lds128(gb + 2 * ((ks * PBB + wn * (NTL / 2) + np) * 32 + lane));
        bf[buf][2 * np] = v.x;
        bf[buf][2 * np + 1] = v.y;
      }
    };
    load_frags(0, 0);
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      if (ks + 1 < KS) load_frags((ks + 1) & 1, ks + 1);
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NTL; ++j) dmma(acc[i][j][0], acc[i][j][1], af[ks & 1][i], bf[ks & 1][j]);
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (++s == S) { s = 0; ph ^= 1u; }
    if (fl & 2) {  // this split's partial tile
      const int split = item / tiles, t = item - split * tiles;
      const int tm = t / P.tilesN, tn = t - tm * P.tilesN;
      double* Cb = P.C + split * P.split_stride;
#pragma unroll
      for (int i = 0; i < MT; ++i) {
        const int64_t row = (int64_t)tm * BMT + wm * WTM + i * 8 + cl;
#pragma unroll
        for (int j = 0; j < NTL; ++j) {
          const int col = tn * BN + wn * WTN + j * 8 + 2 * r4;
          *reinterpret_cast<double2*>(Cb + row * P.ldc + col) = make_double2(acc[i][j][0], acc[i][j][1]);
        }
      }
    }
  }
}

// Fixed-order split reduction with many splits over a small output (small problems split the
// individuals over every SM): CTA = 32 element pairs x 8 groups of consecutive splits; each group
// sums its splits in order, then the 8 group sums are added in group order (deterministic).
constexpr int kRedGroups = 8;
__global__ void __launch_bounds__(256) k_reduce_splits_wide(double* __restrict__ dst, const double* __restrict__ src,
                                                            int64_t n, int S, int64_t stride) {
  __shared__ double2 part[kRedGroups][32];
  const int j = threadIdx.x & 31, g = threadIdx.x >> 5;
  const int64_t e = ((int64_t)blockIdx.x * 32 + j) * 2;
  const int s0 = g * S / kRedGroups, s1 = (g + 1) * S / kRedGroups;
  double2 acc = make_double2(0.0, 0.0);
  if (e < n) {
    int s = s0;
    for (; s + 4 <= s1; s += 4) {  // 4 loads in flight, added in split order
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = *reinterpret_cast<const double2*>(src + (s + u) * stride + e);
#pragma unroll
      for (int u = 0; u < 4; ++u) { acc.x += v[u].x; acc.y += v[u].y; }
    }
    for (; s < s1; ++s) {
      const double2 v = *reinterpret_cast<const double2*>(src + s * stride + e);
      acc.x += v.x;
      acc.y += v.y;
    }
  }
  part[g][j] = acc;
  __syncthreads();
  if (g == 0 && e < n) {
    double2 t = part[0][j];
    for (int h = 1; h < kRedGroups; ++h) { t.x += part[h][j].x; t.y += part[h][j].y; }
    *reinterpret_cast<double2*>(dst + e) = t;
  }
}

// Fixed-order split reduction: dst[e] = sum_s src[s * stride + e]  (stride even).
__global__ void k_reduce_splits(double* __restrict__ dst, const double* __restrict__ src, int64_t n,
                                int S, int64_t stride) {
  for (int64_t e = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) * 2; e < n;
       e += (int64_t)gridDim.x * blockDim.x * 2) {
    if (e + 1 < n) {
      double2 acc = *reinterpret_cast<const double2*>(src + e);
      for (int s = 1; s < S; ++s) {
        const double2 v = *reinterpret_cast<const double2*>(src + s * stride + e);
        acc.x += v.x;
        acc.y += v.y;
      }
      *reinterpret_cast<double2*>(dst + e) = acc;
    } else {
      double acc = src[e];
      for (int s = 1; s < S; ++s) acc += src[s * stride + e];
      dst[e] = acc;
    }
  }
}

// J3: T_k = sum_i P_ik e_ik f_ik^T per alternative k, on DMMA.
// e = [x~_i (q; absent for k = 0), z_ik (d), y_ik (f)] (E rows), f = [z_ik (d), y_ik (f)] (F cols).
// A CTA's 8 warps take 8 consecutive alternatives over the same individuals (the x~ rows are shared
// through L1); a warp owns a 64 x 32 panel of T_k (MT x NT 8x8 DMMA blocks) and loads its fragment
// elements straight from the packed rows (A = P_ik e_ik, B = f_ik, inner dimension = individuals).
// Item = (alternative group, e-panel, f-panel, split); split partials are reduced in fixed order.
// Same-alternative terms T_k[e][f] = sum_i P_ik s_e(i, k) t_f(i, k) with s = [x~_i | z_ik | y_ik]
// (the x~ part absent for alternative 0) and t = [z_ik | y_ik] (the arrow of the block
// structure). CTA = 8 alternatives (one warp each) x an (e, f) tile x a range of individuals.
// Per chunk of CI individuals the rows every warp needs are staged once in shared memory by
// cp.async (16-byte pieces where aligned, double-buffered, zero-filled beyond N / K):
// row i = [x~_i (q, padded to even) | P_i,k0..k0+7 | z_i,k0..k0+7 (8d) | y_i,k0..k0+7 (8f) | 0],
// stride RS = 4 (mod 16) doubles so the 4-row x 8-column fragment gathers are conflict free.
// Each warp builds its fragments from smem; P_ik scales the (narrower) t side.
__host__ __device__ inline int arrow_qe(int q) { return (q + 1) & ~1; }
__host__ __device__ inline int arrow_row_len(int q, int d, int f) { return arrow_qe(q) + 8 + 8 * d + 8 * f + 1; }

template <int MT, int NT>
__global__ void __launch_bounds__(256) k_arrow(int64_t N, int K, int q, int d, int f, int splits, int64_t Npad,
                                               int n_ep, int n_fp, int CI, int RS, const double* __restrict__ Pr,
                                               int ldP, const double* __restrict__ Xp, int ldX,
                                               const double* __restrict__ Zp, int ldZ,
                                               const double* __restrict__ Y, double* Tpart, int64_t tstride) {
  extern __shared__ __align__(16) double sst[];  // [2][CI][RS]
  const int E = q + d + f, F = d + f, RL = arrow_row_len(q, d, f), qe = arrow_qe(q);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n_kg = (K + 7) / 8;
  int item = blockIdx.x;
  const int kg = item % n_kg; item /= n_kg;
  const int ep = item % n_ep; item /= n_ep;
  const int fp = item % n_fp; item /= n_fp;
  const int split = item;
  const int k0 = kg * 8, k = k0 + w;
  const int64_t nch = Npad / CI;
  const int64_t c_begin = split * nch / splits, c_end = (split + 1) * nch / splits;
  const int r4 = lane & 3, c8 = lane >> 2;
  const int oP = qe, oZ = qe + 8, oY = qe + 8 + 8 * d, o0 = RL - 1;  // o0: a zero
  int eoff[MT];
#pragma unroll
  for (int mb = 0; mb < MT; ++mb) {
    const int e = ep * MT * 8 + mb * 8 + c8;
    if (e < q) eoff[mb] = (k == 0) ? o0 : e;
    else if (e < q + d) eoff[mb] = oZ + w * d + (e - q);
    else if (e < E) eoff[mb] = oY + w * f + (e - q - d);
    else eoff[mb] = o0;
  }
  int foff[NT];
#pragma unroll
  for (int nb = 0; nb < NT; ++nb) {
    const int fi = fp * NT * 8 + nb * 8 + c8;
    foff[nb] = fi < d ? oZ + w * d + fi : (fi < F ? oY + w * f + (fi - d) : o0);
  }
  for (int r = threadIdx.x; r < 2 * CI; r += blockDim.x) sst[(size_t)r * RS + o0] = 0.0;  // never staged
  auto cp8 = [](double* dst, const double* src, bool ok) {  // zero-fill when !ok
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(ok ? 8 : 0)
                 : "memory");
  };
  auto cp16 = [](double* dst, const double* src, int bytes) {  // bytes in {0, 8, 16}; rest zero-filled
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes)
                 : "memory");
  };
  const int nz = min(8, K - k0) * d, ny = min(8, K - k0) * f;  // this group's z / y values per row
  const bool y16 = (f % 2) == 0 && (reinterpret_cast<uintptr_t>(Y) & 15) == 0;
  auto stage = [&](int64_t c, int buf) {  // warp per row, lanes across each segment
    double* base = sst + (size_t)buf * CI * RS;
    for (int r = w; r < CI; r += 8) {
      const int64_t i = c * CI + r;
      double* row = base + (size_t)r * RS;
      const double* xr = Xp + i * ldX;  // ldX >= qe: the pair read past an odd q stays in the row
      for (int t = 2 * lane; t < qe; t += 64) cp16(row + t, xr + t, 16);
      if (lane < 4) cp16(row + oP + 2 * lane, Pr + i * ldP + k0 + 2 * lane,
                         8 * max(0, min(2, K - (k0 + 2 * lane))));
      const double* zr = Zp + i * ldZ + k0 * d;
      for (int t = 2 * lane; t < 8 * d; t += 64) cp16(row + oZ + t, zr + (t < nz ? t : 0), 8 * max(0, min(2, nz - t)));
      const double* yr = Y + ((i < N ? i : 0) * K + k0) * f;
      if (y16) {
        for (int t = 2 * lane; t < 8 * f; t += 64)
          cp16(row + oY + t, yr + (t < ny ? t : 0), i < N ? 8 * max(0, min(2, ny - t)) : 0);
      } else {
        for (int t = lane; t < 8 * f; t += 32) cp8(row + oY + t, yr + (t < ny ? t : 0), i < N && t < ny);
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  double acc[MT][NT][2];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NT; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  if (c_begin < c_end) stage(c_begin, 0);
  int buf = 0;
  for (int64_t c = c_begin; c < c_end; ++c, buf ^= 1) {
    if (c + 1 < c_end) stage(c + 1, buf ^ 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncthreads();
    if (k < K) {
      const double* base = sst + (size_t)buf * CI * RS;
#pragma unroll 2
      for (int qq = 0; qq < CI / 4; ++qq) {
        const double* row = base + (size_t)(4 * qq + r4) * RS;
        const double pk = row[oP + w];
        double av[MT], bv[NT];
#pragma unroll
        for (int mb = 0; mb < MT; ++mb) av[mb] = row[eoff[mb]];
#pragma unroll
        for (int nb = 0; nb < NT; ++nb) bv[nb] = pk * row[foff[nb]];
#pragma unroll
        for (int mb = 0; mb < MT; ++mb)
#pragma unroll
          for (int nb = 0; nb < NT; ++nb)
            asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                : "+d"(acc[mb][nb][0]), "+d"(acc[mb][nb][1])
                : "d"(av[mb]), "d"(bv[nb]));
      }
    }
    __syncthreads();  // done with buf before it is refilled
  }
  if (k >= K) return;
  double* out = Tpart + split * tstride + (int64_t)k * E * F;
#pragma unroll
  for (int mb = 0; mb < MT; ++mb) {
    const int e = ep * MT * 8 + mb * 8 + c8;
#pragma unroll
    for (int nb = 0; nb < NT; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int fi = fp * NT * 8 + nb * 8 + 2 * r4 + h;
        if (e < E && fi < F) out[e * F + fi] = acc[mb][nb][h];
      }
  }
}

struct AsmArgs {
  int K, q, d, f, n_beta, off_gamma, n_p;
  const double* C1;  // [pairs_pad][ld1]  (reduced) vech columns [0, n1a)
  int ld1;
  const double* C1b; // [pairs_pad][ld1b] vech columns [n1a, ...)
  int ld1b, n1a;
  const double* C2;  // [n_p_pad][ld2]    (reduced) Z/Y columns [0, n2a)
  int ld2;
  const double* C2b; // [n_p_pad][ld2b]   Z/Y columns [n2a, ...)
  int ld2b, n2a;
  const double* T;   // [K][E][F]         (reduced)
  double* out;
  int ld_out;        // < 0: out is the packed upper triangle (row r: columns r..n_p-1)
  double sign;
};

__device__ __forceinline__ int64_t tri_index(int i, int j, int n) {  // i <= j < n, row-major upper
  return (int64_t)i * n - (int64_t)i * (i - 1) / 2 + (j - i);
}

__global__ void __launch_bounds__(256) k_assemble(const AsmArgs A) {
  const int n_p = A.n_p, q = A.q, d = A.d, f = A.f;
  const int E = q + d + f, F = d + f;
  const int M = A.K - 1;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < (int64_t)n_p * n_p;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int r = (int)(e / n_p), c = (int)(e - (int64_t)r * n_p);
    if (A.ld_out < 0 && c < r) continue;
    double negH;
    if (r < A.n_beta && c < A.n_beta) {
      int k1 = r / q, a1 = r - k1 * q, k2 = c / q, a2 = c - k2 * q;  // 0-based k-1
      const int kl = min(k1, k2), kh = max(k1, k2), al = min(a1, a2), ah = max(a1, a2);
      const int64_t pr = tri_index(kl, kh, M);
      const int v = (int)tri_index(al, ah, q);
      negH = v < A.n1a ? A.C1[pr * A.ld1 + v] : A.C1b[pr * A.ld1b + (v - A.n1a)];
    } else {
      const int lo = min(r, c), hi = max(r, c);
      const int c2 = hi - A.n_beta;
      double u = c2 < A.n2a ? A.C2[(int64_t)lo * A.ld2 + c2] : A.C2b[(int64_t)lo * A.ld2b + (c2 - A.n2a)];
      // same-alternative / generic terms T (J3)
      double tv = 0.0;
      auto cls = [&](int x, int& kind, int& k, int& idx) {
        if (x < A.n_beta) { kind = 0; k = x / q + 1; idx = x - (k - 1) * q; }
        else if (x < A.off_gamma) { kind = 1; k = (x - A.n_beta) / d; idx = x - A.n_beta - k * d; }
        else { kind = 2; k = -1; idx = x - A.off_gamma; }
      };
      int kl, kkl, il, kh, kkh, ih;
      cls(lo, kl, kkl, il);
      cls(hi, kh, kkh, ih);
      // e-index of the row factor, f-index of the column factor (hi is alpha or gamma)
      const int fi = (kh == 1) ? ih : d + ih;
      if (kl == 2) {  // gamma-gamma: sum over alternatives
        for (int k = 0; k < A.K; ++k) tv += A.T[((int64_t)k * E + q + d + il) * F + fi];
      } else if (kh == 2) {  // beta/alpha x gamma: alternative of lo
        const int ei = (kl == 0) ? il : q + il;
        tv = A.T[((int64_t)kkl * E + ei) * F + fi];
      } else if (kkl == kkh) {  // beta/alpha x alpha of the same alternative
        if (kl == 0) tv = A.T[((int64_t)kkl * E + il) * F + fi];
        else {
          const int x = min(il, ih), y = max(il, ih);
          tv = A.T[((int64_t)kkl * E + q + x) * F + y];
        }
      }
      negH = tv - u;
    }
    const int64_t o = A.ld_out < 0 ? (int64_t)r * n_p - (int64_t)r * (r - 1) / 2 + (c - r) : (int64_t)r * A.ld_out + c;
    A.out[o] = -A.sign * negH;
  }
}

// ---- small problems (n_p <= 64): the whole Hessian in one launch --------------------------------
// For a handful of parameters the three GEMMs above are latency: seven launches, split partials and
// an assembly for a few hundred entries (c1: n_p = 18). Here every thread owns <= kSmallEpt entries
// (r <= c) of -H and accumulates, individual by individual, the J-form of P:378-382 / App. B with the
// Jacobian's sparsity written out: with m_r the value of column r in its own alternative's
// utility (x~_ia for beta_k, z_ikc for alpha_k) and u_r = sum_k P_ik J_i[k][r] (P_ik m_r; ybar_ie
// for gamma_e),
//   -H_i[r][c] = [alt(r) = alt(c)] P_i,alt m_r m_c          (beta / alpha x beta / alpha)
//              + P_i,alt(r) m_r y_i,alt(r),e                 (beta / alpha x gamma_e)
//              + sum_k P_ik y_ike y_ike'                     (gamma_e x gamma_e')
//              - u_r u_c.
// CTA partials go to global scratch and the last CTA to finish sums them in CTA order (fixed order:
// deterministic) into the caller's layout.
constexpr int kSmallEpt = 9;     // entries per thread: 256 x 9 >= 64 x 65 / 2
constexpr int kSmallTI = 16;     // individuals per staged tile
constexpr int kSmallMaxKF = 128; // K f of a staged Y row (static shared memory < 48 KB)
struct SmallArgs {
  int64_t N;
  int K, q, d, f, n_p, n_beta, off_gamma;
  const double* Pr; int ldP;
  const double* Xp; int ldX;
  const double* Zp; int ldZ;
  const double* Y;
  double* part;  // [gridDim.x][vech]
  unsigned* counter;
  double* out;
  int ld_out;    // < 0: packed upper triangle
  double sign;
};

__global__ void __launch_bounds__(256) k_hess_small(const SmallArgs A) {
  __shared__ double Ps[kSmallTI][65], Us[kSmallTI][64], Ms[kSmallTI][64];
  __shared__ double Ys[kSmallTI][kSmallMaxKF];
  __shared__ bool last;
  const int tid = threadIdx.x, n = A.n_p, K = A.K, q = A.q, d = A.d, f = A.f;
  const int V = n * (n + 1) / 2;
  // column r -> (kind 0 beta / 1 alpha / 2 gamma, alternative, component)
  auto cls = [&](int x, int& kind, int& k, int& idx) {
    if (x < A.n_beta) { kind = 0; k = x / q + 1; idx = x - (k - 1) * q; }
    else if (x < A.off_gamma) { kind = 1; k = (x - A.n_beta) / d; idx = x - A.n_beta - k * d; }
    else { kind = 2; k = -1; idx = x - A.off_gamma; }
  };
  // this thread's entries j = tid + 256 t (row-major upper triangle order)
  int er[kSmallEpt], ec[kSmallEpt];
  double acc[kSmallEpt];
#pragma unroll
  for (int t = 0; t < kSmallEpt; ++t) {
    acc[t] = 0.0;
    er[t] = ec[t] = -1;
    int j = tid + 256 * t;
    if (j < V) {
      int r = 0;
      while (j >= n - r) { j -= n - r; ++r; }
      er[t] = r;
      ec[t] = r + j;
    }
  }
  const int64_t ntiles = (A.N + kSmallTI - 1) / kSmallTI;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i0 = tile * kSmallTI;
    const int nt = (int)(A.N - i0 < kSmallTI ? A.N - i0 : kSmallTI);
    __syncthreads();  // the previous tile's readers are done
    // staging: read-only loads, unrolled so that each thread's loads are in flight together (one
    // memory round trip per tile, not one per element)
#pragma unroll 4
    for (int e = tid; e < nt * K; e += 256) {
      const int ii = e / K, k = e - ii * K;
      Ps[ii][k] = __ldg(A.Pr + (i0 + ii) * A.ldP + k);
    }
#pragma unroll 4
    for (int e = tid; e < nt * K * f; e += 256) {
      const int ii = e / (K * f), o = e - ii * (K * f);
      Ys[ii][o] = __ldg(A.Y + (i0 + ii) * (int64_t)(K * f) + o);
    }
#pragma unroll 4
    for (int e = tid; e < nt * n; e += 256) {
      const int ii = e / n, r = e - ii * n;
      const int64_t i = i0 + ii;
      int kind, k, idx;
      cls(r, kind, k, idx);
      const double P = __ldg(A.Pr + i * A.ldP + (kind == 2 ? K + idx : k));  // ybar_ie for gamma_e
      const double m = kind == 0 ? __ldg(A.Xp + i * A.ldX + idx) : (kind == 1 ? __ldg(A.Zp + i * A.ldZ + k * d + idx) : 1.0);
      Ms[ii][r] = m;
      Us[ii][r] = P * m;
    }
    __syncthreads();
#pragma unroll
    for (int t = 0; t < kSmallEpt; ++t) {
      if (er[t] < 0) continue;
      const int r = er[t], c = ec[t];
      int kr, ar, ir, kc, ac, ic;
      cls(r, kr, ar, ir);
      cls(c, kc, ac, ic);
      double s = 0.0;
      for (int ii = 0; ii < nt; ++ii) {
        double v = -Us[ii][r] * Us[ii][c];
        if (kr != 2 && kc != 2) {
          if (ar == ac) v = fma(Ps[ii][ar] * Ms[ii][r], Ms[ii][c], v);
        } else if (kr != 2) {  // c is gamma_ic (r < c: gamma columns come last)
          v = fma(Ps[ii][ar] * Ms[ii][r], Ys[ii][ar * f + ic], v);
        } else {
          for (int k = 0; k < K; ++k) v = fma(Ps[ii][k] * Ys[ii][k * f + ir], Ys[ii][k * f + ic], v);
        }
        s += v;
      }
      acc[t] += s;
    }
  }
  double* my = A.part + (size_t)blockIdx.x * V;
#pragma unroll
  for (int t = 0; t < kSmallEpt; ++t)
    if (er[t] >= 0) my[tid + 256 * t] = acc[t];
  __threadfence();
  __syncthreads();
  if (tid == 0) last = (atomicAdd(A.counter, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
#pragma unroll
  for (int t = 0; t < kSmallEpt; ++t) {
    if (er[t] < 0) continue;
    const int j = tid + 256 * t, r = er[t], c = ec[t];
    double s = 0.0;
    int b = 0;
    for (; b + 8 <= (int)gridDim.x; b += 8) {  // 8 loads in flight, summed in CTA order
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = __ldcg(A.part + (size_t)(b + u) * V + j);
#pragma unroll
      for (int u = 0; u < 8; ++u) s += v[u];
    }
    for (; b < (int)gridDim.x; ++b) s += __ldcg(A.part + (size_t)b * V + j);
    const double v = -A.sign * s;  // s = -H[r][c]
    if (A.ld_out < 0) {
      A.out[j] = v;  // row-major upper triangle: j is the packed index
    } else {
      A.out[(int64_t)r * A.ld_out + c] = v;
      A.out[(int64_t)c * A.ld_out + r] = v;
    }
  }
  if (tid == 0) *A.counter = 0u;
}

}  // namespace

// ------------------------------------------------------------------------------------------
// Host plan
// ------------------------------------------------------------------------------------------

struct GemmJob {
  int BN, KC, nwarp = 8, nraw = 2;
  // Operand materialisation (k_frag): mat_b alone -> k_gen_gemm<..., BPRE> generates only A;
  // mat_a && mat_b -> k_pipe_gemm (pure TMA/mbarrier pipeline). b_design: B depends only on the
  // packed design rows (J1's x~_a x~_b), so it is rebuilt only after a re-pack.
  bool mat_a = false, mat_b = false, b_design = false;
  bool own_afrag = true;   // false: afrag borrowed from j1 (the J1 tail job shares j1's weights)
  double* afrag = nullptr;  // [tilesM][nchunks][GA_D]
  double* bfrag = nullptr;  // [tilesN][nchunks][GB_D]
  int dnseg = 0, dseg_id[3] = {0, 0, 0};  // stage layout the descriptors were built against
  bool agen = true;  // A operand uses the general generator form (J1)
  int BM = mnl::BM;  // M-tile height: 128, or 64 for a pipelined J1 with few weight pairs
  int MA, MB, tilesM, tilesN, splits;
  // N-slabs (k_pipe_gemm jobs whose whole-N operands do not fit): the fragment buffers hold
  // slab_chunks chunks; the operands are materialised and consumed one slab at a time, each slab
  // writing its own split partials (nslab x splits, reduced in a fixed order)
  int64_t slab_chunks = 0;
  int nslab = 1;
  int skip_off = -1;  // GemmParams::skip_off
  int64_t nchunks;
  ColDesc* dA = nullptr;  // device
  ColDesc* dB = nullptr;
  double* Cpart = nullptr;  // [splits][tilesM*128][tilesN*BN]
  double* Cred = nullptr;   // [tilesM*128][tilesN*BN]
  int ldc;
  int64_t split_stride;
  int nseg;
  int seg_id[3];
  int stage_doubles;
  size_t smem;
};

struct HessPlan {
  bool small = false;  // n_p <= 64: k_hess_small, one launch (nothing below is used)
  int small_grid = 0;
  double* small_part = nullptr;
  bool has_j2;
  bool has_j2b = false;  // J2's Z/Y columns as whole main tiles + a narrow tail job (shares j2's A)
  int n2a = 0;           // Z/Y columns computed by j2
  bool bvalid = false;  // J1's precomputed B fragments match the packed design rows
  GemmJob j1, j1b, j2, j2b;  // j1b / j2b: the columns beyond the last whole main tile of j1 / j2
  bool has_j1b = false;
  int n1a = 0;          // vech columns computed by j1
  int ar_splits, ar_mt, ar_nt, ar_ep, ar_fp, ar_ci, ar_rs;
  double* Tpart = nullptr;
  double* T = nullptr;
  unsigned* counters = nullptr;  // [2]
  cudaEvent_t ev[8] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // [7]: before operand prep
  size_t bytes = 0;
  int sms;
};

constexpr size_t kFragSmemMax = 220 * 1024;  // k_frag's staged rows
// k_frag stages KC / nh rows per CTA (nh | KC / 4): the smallest nh keeping the stage <= 48 KB
// (occupancy), else the smallest that fits at all; 0 if none does
static int frag_nh(size_t stage_doubles) {
  for (int nh = 1; nh <= 8; nh *= 2)
    if (stage_doubles * sizeof(double) / nh <= 48 * 1024) return nh;
  for (int nh = 1; nh <= 8; nh *= 2)
    if (stage_doubles * sizeof(double) / nh <= kFragSmemMax) return nh;
  return 0;
}

static int choose_splits(int tiles, int64_t nchunks, int sms, int min_chunks) {
  int best = 1;
  double best_eff = -1.0;
  for (int S = 1; S <= 256; ++S) {
    if (nchunks / S < min_chunks && S > 1) break;
    const int64_t items = (int64_t)tiles * S;
    const int64_t waves = (items + sms - 1) / sms;
    const double eff = (double)items / (double)(waves * sms);
    if (eff > best_eff + 1e-9) { best_eff = eff; best = S; }
    if (eff > 0.995) break;
  }
  return best;
}

// Output-tile width: the widest of {128, 96, 64} whose padded width is within 5% of the smallest
// padded width (wider tiles reuse each generated operand more; measured equal time on c4 for
// 128 vs 96).
static int choose_bn(int MB) {
  int64_t min_pad = -1;
  for (int bn : {128, 96, 64}) {
    const int64_t pad = (int64_t)(MB + bn - 1) / bn * bn;
    if (min_pad < 0 || pad < min_pad) min_pad = pad;
  }
  for (int bn : {128, 96, 64})
    if ((double)((MB + bn - 1) / bn * bn) <= 1.05 * (double)min_pad) return bn;
  return 64;
}

static bool setup_job(GemmJob& J, const std::vector<ColDesc>& A, const std::vector<ColDesc>& B, int BN,
                      int KC, const Packed& pk, const int* segs, int nseg, int sms, size_t* bytes,
                      bool pipe = false) {
  J.BN = BN;
  J.KC = KC;
  J.nwarp = 8;
  J.MA = (int)A.size();
  J.MB = (int)B.size();
  J.tilesM = (J.MA + J.BM - 1) / J.BM;
  J.tilesN = (J.MB + BN - 1) / BN;
  J.nchunks = pk.Npad / KC;
  if (J.slab_chunks <= 0 || J.slab_chunks >= J.nchunks) J.slab_chunks = J.nchunks;
  J.nslab = (int)((J.nchunks + J.slab_chunks - 1) / J.slab_chunks);
  J.splits = choose_splits(J.tilesM * J.tilesN, J.slab_chunks, sms, 4);
  J.ldc = J.tilesN * BN;
  J.split_stride = (int64_t)J.tilesM * J.BM * J.ldc;
  J.nseg = nseg;
  int off = 0;
  for (int s = 0; s < nseg; ++s) {
    J.seg_id[s] = segs[s];
    const int ld = segs[s] == 0 ? pk.ldP : (segs[s] == 1 ? pk.ldX : pk.ldZ);
    off += KC * ld;
  }
  J.stage_doubles = off;
  // descriptors padded to whole tiles; padding columns generate exact zeros
  std::vector<ColDesc> hA(A), hB(B);
  ColDesc zero{0, 0, 0, 0, 0.0, 0.0};
  hA.resize((size_t)J.tilesM * J.BM, zero);
  hB.resize((size_t)J.tilesN * BN, zero);
  if (cudaMalloc(&J.dA, hA.size() * sizeof(ColDesc)) != cudaSuccess) return false;
  if (cudaMalloc(&J.dB, hB.size() * sizeof(ColDesc)) != cudaSuccess) return false;
  cudaMemcpy(J.dA, hA.data(), hA.size() * sizeof(ColDesc), cudaMemcpyHostToDevice);
  cudaMemcpy(J.dB, hB.data(), hB.size() * sizeof(ColDesc), cudaMemcpyHostToDevice);
  const size_t cbytes = (size_t)J.split_stride * sizeof(double);
  if (cudaMalloc(&J.Cpart, cbytes * J.splits * J.nslab) != cudaSuccess) return false;
  if (cudaMalloc(&J.Cred, cbytes) != cudaSuccess) return false;
  *bytes += cbytes * (J.splits * J.nslab + 1) + (hA.size() + hB.size()) * sizeof(ColDesc);
  if (pipe) return true;  // k_pipe_gemm: no generator staging
  const size_t lim = 220 * 1024;
  for (J.nraw = 2; J.nraw >= 1; --J.nraw) {  // prefer two raw stages; one if the stage is large
    J.smem = (size_t)(2 * (KC / 4) * 8 * 64 + 2 * (KC / 4) * (BN / 16) * 64 + J.nraw * J.stage_doubles) *
             sizeof(double);
    if (J.smem <= lim) return true;
  }
  J.nraw = 1;
  return false;
}

static void free_job(GemmJob& J) {
  cudaFree(J.dA);
  cudaFree(J.dB);
  cudaFree(J.bfrag);
  if (J.own_afrag) cudaFree(J.afrag);
  J.own_afrag = true;
  J.afrag = J.bfrag = nullptr;
  J.mat_a = J.mat_b = J.b_design = false;
  cudaFree(J.Cpart);
  cudaFree(J.Cred);
  J.dA = J.dB = nullptr;
  J.Cpart = J.Cred = nullptr;
}

// Fragment buffer of `tiles` operand tiles (128 rows for A, BN for B) over all chunks, if it fits
// with 4 GB of HBM to spare (otherwise the operand stays generated in-kernel).
static double* alloc_frag(int tiles, int width, const Packed& pk, size_t* bytes) {
  const size_t fb = (size_t)tiles * width * (size_t)pk.Npad * sizeof(double);
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  if (getenv("MNL_NO_MATERIALISE") || fb > ((size_t)48 << 30) || fb + ((size_t)4 << 30) >= free_b) return nullptr;
  double* p = nullptr;
  if (cudaMalloc(&p, fb) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  *bytes += fb;
  return p;
}

// Fragment buffer of `tiles` operand tiles over `chunks` chunks of KC individuals (an N-slab).
static double* alloc_frag_chunks(int tiles, int width, int64_t chunks, int KC, size_t* bytes) {
  const size_t fb = (size_t)tiles * width * (size_t)chunks * KC * sizeof(double);
  double* p = nullptr;
  if (cudaMalloc(&p, fb) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  *bytes += fb;
  return p;
}

// Chunks per N-slab for materialised operands of `per_chunk` bytes per chunk: all of them when they
// fit in min(48 GB, free - 4 GB), else the balanced slab size under that budget; 0 when even a
// 64-chunk slab does not fit (the operands are then generated in-kernel). MNL_FRAG_SLAB_CHUNKS
// forces a slab size (tests of the slabbed path at small N).
static int64_t frag_slab_chunks(size_t per_chunk, int64_t nch) {
  if (const char* e = getenv("MNL_FRAG_SLAB_CHUNKS")) {
    const int64_t f = atoll(e);
    if (f > 0) return std::min<int64_t>(f, nch);
  }
  if (getenv("MNL_NO_MATERIALISE")) return 0;
  size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);
  const size_t reserve = (size_t)4 << 30, cap = (size_t)48 << 30;
  const size_t budget = std::min(cap, free_b > reserve ? free_b - reserve : (size_t)0);
  const int64_t fit = (int64_t)(budget / per_chunk);
  if (fit >= nch) return nch;
  if (fit < 64) return 0;
  const int64_t nslab = (nch + fit - 1) / fit;
  return (nch + nslab - 1) / nslab;
}

// Tile widths of the 64-row k_pipe_gemm: the widest of {128, 96, 64} within 5 % of the smallest padding.
static int choose_bn_pipe64(int MB) {
  int64_t min_pad = -1;
  for (int bn : {128, 96, 64}) {
    const int64_t pad = (int64_t)(MB + bn - 1) / bn * bn;
    if (min_pad < 0 || pad < min_pad) min_pad = pad;
  }
  for (int bn : {128, 96, 64})
    if ((double)((MB + bn - 1) / bn * bn) <= 1.05 * (double)min_pad) return bn;
  return 64;
}

// Tile widths k_pipe_gemm is instantiated for: the widest of {128, 112, 96, 64, 48} within 5% of the
// smallest padded width.
static int choose_bn_pipe(int MB) {
  int64_t min_pad = -1;
  for (int bn : {128, 112, 96, 64, 48}) {
    const int64_t pad = (int64_t)(MB + bn - 1) / bn * bn;
    if (min_pad < 0 || pad < min_pad) min_pad = pad;
  }
  for (int bn : {128, 112, 96, 64, 48})
    if ((double)((MB + bn - 1) / bn * bn) <= 1.05 * (double)min_pad) return bn;
  return 48;
}

// k_hess_small serves problems whose Hessian is a few hundred to ~2000 entries and whose direct
// per-individual work (N x vech x a few FMAs, + K per gamma-gamma entry) is small: there one launch
// beats the GEMM pipeline's seven. MNL_NO_SMALL forces the general path (tests).
static bool small_ok(const Dims& D) {
  if (D.n_p > 64 || D.K > 65 || (int64_t)D.K * D.f > kSmallMaxKF || getenv("MNL_NO_SMALL")) return false;
  const double V = D.n_p * (D.n_p + 1) / 2.0, G = D.f * (D.f + 1) / 2.0;
  return (double)D.N * (3.0 * V + G * D.K) <= 5e8;
}

HessPlan* hess_plan_create(const Dims& D, const Packed& pk, int sms) {
  HessPlan* hp = new HessPlan();
  hp->sms = sms;
  const int K = D.K, q = D.q, d = D.d, f = D.f;
  if (small_ok(D)) {
    hp->small = true;
    hp->small_grid = (int)std::max<int64_t>(1, std::min<int64_t>(sms, (D.N + kSmallTI - 1) / kSmallTI));
    const size_t vb = (size_t)D.n_p * (D.n_p + 1) / 2 * sizeof(double);
    bool ok = cudaMalloc(&hp->small_part, vb * hp->small_grid) == cudaSuccess &&
              cudaMalloc(&hp->counters, 2 * sizeof(unsigned)) == cudaSuccess &&
              cudaMemset(hp->counters, 0, 2 * sizeof(unsigned)) == cudaSuccess;
    for (auto& e : hp->ev) cudaEventCreate(&e);
    hp->bytes = vb * hp->small_grid;
    if (!ok) {
      hess_plan_destroy(hp);
      return nullptr;
    }
    return hp;
  }
  // stage layouts: segment 0 = Pr, 1 = Xp, 2 = Zp; offsets are set per job below
  auto seg_ld = [&](int s) { return s == 0 ? pk.ldP : (s == 1 ? pk.ldX : pk.ldZ); };
  bool ok = true;
  size_t bytes = 0;
  {  // J1: pairs x vech over Pr + Xp
    const int segs[2] = {0, 1};
    for (int KC : {32, 16}) {
      const int offP = 0, offX = KC * seg_ld(0);
      std::vector<ColDesc> A, B;
      for (int k = 1; k < K; ++k)
        for (int l = k; l < K; ++l)
          A.push_back(ColDesc{offP + k, pk.ldP, offP + l, pk.ldP, k == l ? 1.0 : 0.0, -1.0});
      for (int a = 0; a < q; ++a)
        for (int b = a; b < q; ++b) B.push_back(ColDesc{offX + a, pk.ldX, offX + b, pk.ldX, 0.0, 1.0});
      // padding columns point at Xp[.][0] (finite) with c0 = s = 0
      // Split the vech columns: whole 128-column tiles in j1, a narrow remainder job j1b (its own
      // width) instead of padding the last tile (c4: 1326 = 10 x 128 + 46; c5: 496 = 3 x 128 + 112).
      const int nv = (int)B.size(), rem = nv % 128;
      const bool split = nv > 128 && rem > 0 && rem <= 112;
      hp->n1a = split ? nv - rem : nv;
      std::vector<ColDesc> Ba(B.begin(), B.begin() + hp->n1a), Bb(B.begin() + hp->n1a, B.end());
      const bool frag_fits = frag_nh((size_t)KC * (pk.ldP + pk.ldX)) > 0;
      // Materialise both operands (k_pipe_gemm) when the per-evaluation write of the weights
      // (8 N 128 tilesM bytes) is small next to the GEMM (~23/vech of it at the measured rates):
      // vech >= 256. Otherwise materialise only the design-only B (once per design) if it fits.
      GemmJob& J = hp->j1;
      const int64_t nch = pk.Npad / KC;
      const bool pipe_ok = KC == 32 && nv >= 256 && frag_fits && !getenv("MNL_NO_PIPE");
      // M-tile height of the pipelined GEMM: 64 when it pads the weight pairs clearly less than 128
      // (c3: 190 pairs -> 192 rows instead of 256); the tile widths then come from {128, 96, 64}
      const int np = (int)A.size();
      const int bm = (pipe_ok && (np + 63) / 64 * 64 < 0.95 * ((np + 127) / 128 * 128)) ? 64 : BM;
      const int tilesM = (np + bm - 1) / bm;
      int bn1 = split ? 128 : (pipe_ok ? (bm == 64 ? choose_bn_pipe64(nv) : choose_bn_pipe(nv)) : choose_bn(nv));
      const int bnt_p = split ? (bm == 64 ? choose_bn_pipe64(rem) : choose_bn_pipe(rem)) : 0;
      double *af = nullptr, *bf = nullptr, *tbf = nullptr;
      int64_t slab = 0;
      if (pipe_ok) {  // both operands materialised, whole-N or in N-slabs of the same size
        const size_t per_chunk =
            ((size_t)tilesM * bm + (size_t)((hp->n1a + bn1 - 1) / bn1) * bn1 + bnt_p) * KC * sizeof(double);
        slab = frag_slab_chunks(per_chunk, nch);
        if (slab > 0) {
          af = alloc_frag_chunks(tilesM, bm, slab, KC, &bytes);
          bf = af ? alloc_frag_chunks((hp->n1a + bn1 - 1) / bn1, bn1, slab, KC, &bytes) : nullptr;
          tbf = (bf && split) ? alloc_frag_chunks(1, bnt_p, slab, KC, &bytes) : nullptr;
          if (!bf || (split && !tbf)) {
            cudaFree(af);
            cudaFree(bf);
            cudaFree(tbf);
            af = bf = tbf = nullptr;
          }
        }
      }
      if (!af) {  // weights generated in-kernel; the design-only B materialised whole if it fits
        slab = 0;
        if (!split) bn1 = choose_bn(nv);
        bf = frag_fits ? alloc_frag((hp->n1a + bn1 - 1) / bn1, bn1, pk, &bytes) : nullptr;
      }
      J.afrag = af;
      J.bfrag = bf;
      J.own_afrag = true;
      J.BM = af ? bm : BM;  // in-kernel generation (k_gen_gemm) is built for 128-row tiles
      J.mat_a = af != nullptr;
      J.mat_b = bf != nullptr;
      J.slab_chunks = slab;
      J.b_design = slab == 0 || slab >= nch;  // B cached across evaluations only when whole-N
      J.dnseg = 2;
      J.dseg_id[0] = 0;
      J.dseg_id[1] = 1;
      const int segs_p[1] = {0};  // k_gen_gemm<..., BPRE> stages only the probabilities
      const bool bonly = J.mat_b && !J.mat_a;
      bool good = setup_job(J, A, Ba, bn1, KC, pk, bonly ? segs_p : segs, bonly ? 1 : 2, sms, &bytes, J.mat_a);
      hp->has_j1b = split;
      if (good && split) {
        GemmJob& T = hp->j1b;
        const int bnt = J.mat_a ? bnt_p : choose_bn(rem);
        T.bfrag = tbf;
        T.afrag = tbf ? J.afrag : nullptr;  // the tail shares j1's weights (slab by slab)
        T.own_afrag = tbf == nullptr;
        T.mat_a = T.mat_b = tbf != nullptr;
        T.slab_chunks = J.slab_chunks;
        T.b_design = J.b_design;
        T.BM = T.mat_a ? J.BM : BM;  // reads j1's weight fragments
        T.dnseg = 2;
        T.dseg_id[0] = 0;
        T.dseg_id[1] = 1;
        good = setup_job(T, A, Bb, bnt, KC, pk, segs, 2, sms, &bytes, T.mat_a);
      }
      if (good) break;
      free_job(hp->j1);
      free_job(hp->j1b);
      if (KC == 16) ok = false;
    }
  }
  hp->has_j2 = (d + f) > 0;
  if (ok && hp->has_j2) {
    const int segs[3] = {0, 1, 2};
    const int nseg = d > 0 ? 3 : 2;
    for (int KC : {32, 16}) {
      const int offP = 0, offX = KC * seg_ld(0), offZ = offX + KC * seg_ld(1);
      std::vector<ColDesc> A, B;
      for (int k = 1; k < K; ++k)
        for (int a = 0; a < q; ++a) A.push_back(ColDesc{offP + k, pk.ldP, offX + a, pk.ldX, 0.0, 1.0});
      std::vector<ColDesc> AG;
      for (int k = 0; k < K; ++k)
        for (int c = 0; c < d; ++c) AG.push_back(ColDesc{offP + k, pk.ldP, offZ + k * d + c, pk.ldZ, 0.0, 1.0});
      for (int e = 0; e < f; ++e) AG.push_back(ColDesc{offP + K + e, pk.ldP, offX + 0, pk.ldX, 0.0, 1.0});
      A.insert(A.end(), AG.begin(), AG.end());
      B = AG;
      hp->j2.agen = false;
      // both operands depend on the probabilities: materialised per evaluation when the write
      // (8 N (MA + MB) bytes) is small next to the GEMM (23 (1/MA + 1/MB) of it): MB >= 192, MA >= 512
      GemmJob& J = hp->j2;
      const int MA = (int)A.size(), MB = (int)B.size();
      const bool frag_fits = frag_nh((size_t)KC * (pk.ldP + pk.ldX + (d > 0 ? pk.ldZ : 0))) > 0;
      int bn2 = choose_bn(MB);
      hp->has_j2b = false;
      hp->n2a = MB;
      int bnt = 0;  // tail width when split
      if (KC == 32 && MB >= 192 && MA >= 512 && frag_fits && !getenv("MNL_NO_PIPE")) {
        int bnp = choose_bn_pipe(MB);
        // whole main tiles + a narrow tail when that executes fewer columns (c5: 260 = 2 x 112 + 36
        // -> 272 instead of 3 x 96 = 288)
        int best = (MB + bnp - 1) / bnp * bnp;
        for (int bm : {128, 112, 96}) {
          const int main_cols = MB / bm * bm, rem = MB - main_cols;
          if (main_cols == 0 || rem == 0) continue;
          int tail = 0;
          for (int bt : {48, 64, 96, 112, 128})
            if (bt >= rem) { tail = bt; break; }
          if (tail && main_cols + tail < best * 0.98) {
            best = main_cols + tail;
            bnp = bm;
            bnt = tail;
            hp->n2a = main_cols;
          }
        }
        J.afrag = alloc_frag((MA + BM - 1) / BM, BM, pk, &bytes);
        J.bfrag = J.afrag ? alloc_frag((hp->n2a + bnp - 1) / bnp, bnp, pk, &bytes) : nullptr;
        if (J.afrag && !J.bfrag) {
          cudaFree(J.afrag);
          J.afrag = nullptr;
        }
        if (J.bfrag) bn2 = bnp;
        hp->has_j2b = J.bfrag != nullptr && bnt > 0;
        if (!hp->has_j2b) hp->n2a = MB;
      }
      std::vector<ColDesc> Ba(B.begin(), B.begin() + hp->n2a), Bb(B.begin() + hp->n2a, B.end());
      J.own_afrag = true;
      J.mat_a = J.mat_b = J.bfrag != nullptr;
      J.b_design = false;
      J.dnseg = nseg;
      for (int sg = 0; sg < 3; ++sg) J.dseg_id[sg] = segs[sg];
      J.skip_off = (K - 1) * q;  // n_beta: C2 rows are theta indices, columns start at n_beta
      bool good = setup_job(J, A, Ba, bn2, KC, pk, segs, nseg, sms, &bytes, J.mat_a);
      if (good && hp->has_j2b) {
        GemmJob& T = hp->j2b;
        T.agen = false;
        T.bfrag = alloc_frag(1, bnt, pk, &bytes);
        T.afrag = J.afrag;  // the tail shares j2's A operand (materialised by j2's k_frag launch)
        T.own_afrag = false;
        T.mat_a = T.mat_b = T.bfrag != nullptr;
        T.b_design = false;
        T.dnseg = nseg;
        for (int sg = 0; sg < 3; ++sg) T.dseg_id[sg] = segs[sg];
        T.skip_off = (K - 1) * q + hp->n2a;  // its columns start at n_beta + n2a
        good = T.bfrag != nullptr && setup_job(T, A, Bb, bnt, KC, pk, segs, nseg, sms, &bytes, true);
        if (!good) free_job(hp->j2b);
      }
      if (good) break;
      free_job(hp->j2);
      hp->has_j2b = false;
      if (KC == 16) ok = false;
    }
    const int E = q + d + f, F = d + f;
    {
      const int mbs = (E + 7) / 8;
      hp->ar_mt = mbs > 6 ? 8 : (mbs > 4 ? 6 : (mbs > 2 ? 4 : 2));
    }
    hp->ar_nt = (F + 7) / 8 > 2 ? 4 : 2;
    hp->ar_ep = (E + hp->ar_mt * 8 - 1) / (hp->ar_mt * 8);
    hp->ar_fp = (F + hp->ar_nt * 8 - 1) / (hp->ar_nt * 8);
    const int base_items = (K + 7) / 8 * hp->ar_ep * hp->ar_fp;
    hp->ar_rs = pad4mod16(arrow_row_len(q, d, f));
    hp->ar_ci = 32;
    while (hp->ar_ci > 4 && (size_t)2 * hp->ar_ci * hp->ar_rs * sizeof(double) > (size_t)200 * 1024) hp->ar_ci /= 2;
    const int64_t nch = pk.Npad / hp->ar_ci;
    // splits of the individuals: minimise the makespan waves(S) / S (the work per item ~ 1 / S) over
    // the resident CTAs (registers allow 2 per SM; shared memory may allow fewer), keeping >= 8
    // chunks per item; the smallest S reaching the minimum (fewest partials to reduce)
    const size_t ar_smem = (size_t)2 * hp->ar_ci * hp->ar_rs * sizeof(double);
    const int per_sm = std::max(1, std::min(2, (int)((size_t)(227 * 1024) / std::max<size_t>(ar_smem, 1))));
    const int64_t slots = (int64_t)sms * per_sm;
    int S = 1;
    double best = 1e30;
    for (int s2 = 1; s2 <= 256 && nch / s2 >= 8; ++s2) {
      const int64_t items = (int64_t)base_items * s2;
      const double span = (double)((items + slots - 1) / slots) / s2;
      if (span < best * (1.0 - 1e-9)) {
        best = span;
        S = s2;
      }
    }
    hp->ar_splits = S;
    const size_t tb = ((size_t)K * E * F + 1) / 2 * 2 * sizeof(double);
    if (cudaMalloc(&hp->Tpart, tb * S) != cudaSuccess) ok = false;
    if (cudaMalloc(&hp->T, tb) != cudaSuccess) ok = false;
    bytes += tb * (S + 1);
  }
  for (auto& e : hp->ev) cudaEventCreate(&e);
  if (cudaMalloc(&hp->counters, 2 * sizeof(unsigned)) != cudaSuccess) ok = false;
  else cudaMemset(hp->counters, 0, 2 * sizeof(unsigned));
  hp->bytes = bytes;
  if (!ok) {
    hess_plan_destroy(hp);
    return nullptr;
  }
  return hp;
}

void hess_plan_destroy(HessPlan* hp) {
  if (!hp) return;
  free_job(hp->j1);
  free_job(hp->j1b);
  free_job(hp->j2);
  free_job(hp->j2b);
  cudaFree(hp->Tpart);
  cudaFree(hp->T);
  cudaFree(hp->small_part);
  cudaFree(hp->counters);
  for (auto& e : hp->ev)
    if (e) cudaEventDestroy(e);
  delete hp;
}

size_t hess_plan_bytes(const HessPlan* hp) { return hp ? hp->bytes : 0; }

template <int BN, int KC, int NWARP, bool AGEN, bool BPRE = false>
static cudaError_t run_gemm(const GemmJob& J, const Packed& pk, unsigned* counter, int sms, cudaStream_t st) {
  GemmParams P;
  P.descA = J.dA;
  P.descB = J.dB;
  P.tilesM = J.tilesM;
  P.tilesN = J.tilesN;
  P.splits = J.splits;
  P.nchunks = J.nchunks;
  P.cstride = J.nchunks;
  P.C = J.Cpart;
  P.ldc = J.ldc;
  P.split_stride = J.split_stride;
  P.nseg = J.nseg;
  int off = 0;
  for (int s = 0; s < J.nseg; ++s) {
    const int id = J.seg_id[s];
    P.seg_ptr[s] = id == 0 ? pk.Pr : (id == 1 ? pk.Xp : pk.Zp);
    P.seg_ld[s] = id == 0 ? pk.ldP : (id == 1 ? pk.ldX : pk.ldZ);
    P.seg_off[s] = off;
    off += KC * P.seg_ld[s];
  }
  P.stage_doubles = off;
  P.stage_bytes = (unsigned)(off * 8);
  P.nraw = J.nraw;
  P.bfrag = J.bfrag;
  P.counter = counter;
  P.skip_off = J.skip_off;
  static uint64_t attr_mask = 0;
  cudaError_t e = set_once_per_device(attr_mask, [] {
    return cudaFuncSetAttribute(k_gen_gemm<BN, KC, NWARP, AGEN, BPRE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                220 * 1024);
  });
  if (e != cudaSuccess) return e;
  const int items = J.tilesM * J.tilesN * J.splits;
  const int grid = std::min(items, sms * (NWARP < 8 ? 8 / NWARP : 1));
  cudaMemsetAsync(counter, 0, sizeof(unsigned), st);
  k_gen_gemm<BN, KC, NWARP, AGEN, BPRE><<<grid, NWARP * 32, J.smem, st>>>(P);
  count_launch();
  return cudaGetLastError();
}

template <int BN, int BMT = BM>
static cudaError_t run_pipe(const GemmJob& J, unsigned* counter, int sms, cudaStream_t st, int slab) {
  constexpr int KC = 32, S = (200 * 1024) / ((KC / 4) * (BMT / 16 + BN / 16) * 64 * 8);  // stages in ~200 KB
  constexpr size_t smem = (size_t)S * (KC / 4) * (BMT / 16 + BN / 16) * 64 * sizeof(double);
  GemmParams P{};
  P.tilesM = J.tilesM;
  P.tilesN = J.tilesN;
  P.splits = J.splits;
  P.nchunks = std::min<int64_t>(J.slab_chunks, J.nchunks - (int64_t)slab * J.slab_chunks);  // this slab's
  P.cstride = J.slab_chunks;
  P.C = J.Cpart + (size_t)slab * J.splits * J.split_stride;
  P.ldc = J.ldc;
  P.split_stride = J.split_stride;
  P.bfrag = J.bfrag;
  P.counter = counter;
  P.skip_off = J.skip_off;
  static uint64_t attr_mask = 0;
  cudaError_t e = set_once_per_device(attr_mask, [smem] {
    return cudaFuncSetAttribute(k_pipe_gemm<BN, KC, S, BMT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  });
  if (e != cudaSuccess) return e;
  const int items = J.tilesM * J.tilesN * J.splits;
  cudaMemsetAsync(counter, 0, sizeof(unsigned), st);
  k_pipe_gemm<BN, KC, S, BMT><<<std::min(items, sms), 8 * 32 + 32, smem, st>>>(P, J.afrag);
  count_launch();
  return cudaGetLastError();
}

// the GEMM of one job (of its N-slab `slab` when the operands are slabbed), without the reduction
static cudaError_t run_gemm_only(const GemmJob& J, const Packed& pk, unsigned* counter, int sms, cudaStream_t st,
                                 int slab = 0) {
  cudaError_t e;
  if (J.mat_a && J.BM == 64) {
    if (J.BN == 128) e = run_pipe<128, 64>(J, counter, sms, st, slab);
    else if (J.BN == 96) e = run_pipe<96, 64>(J, counter, sms, st, slab);
    else e = run_pipe<64, 64>(J, counter, sms, st, slab);
  } else if (J.mat_a) {
    if (J.BN == 128) e = run_pipe<128>(J, counter, sms, st, slab);
    else if (J.BN == 96) e = run_pipe<96>(J, counter, sms, st, slab);
    else if (J.BN == 112) e = run_pipe<112>(J, counter, sms, st, slab);
    else if (J.BN == 64) e = run_pipe<64>(J, counter, sms, st, slab);
    else e = run_pipe<48>(J, counter, sms, st, slab);
  } else if (J.agen) {  // J1: weights P_k (delta_kl - P_l) x vech(x~ x~^T)
    if (J.BN == 128 && J.mat_b) e = J.KC == 32 ? run_gemm<128, 32, 8, true, true>(J, pk, counter, sms, st) : run_gemm<128, 16, 8, true, true>(J, pk, counter, sms, st);
    else if (J.BN == 128) e = J.KC == 32 ? run_gemm<128, 32, 8, true>(J, pk, counter, sms, st) : run_gemm<128, 16, 8, true>(J, pk, counter, sms, st);
    else if (J.BN == 96 && J.mat_b) e = J.KC == 32 ? run_gemm<96, 32, 8, true, true>(J, pk, counter, sms, st) : run_gemm<96, 16, 8, true, true>(J, pk, counter, sms, st);
    else if (J.BN == 96) e = J.KC == 32 ? run_gemm<96, 32, 8, true>(J, pk, counter, sms, st) : run_gemm<96, 16, 8, true>(J, pk, counter, sms, st);
    else if (J.mat_b) e = J.KC == 32 ? run_gemm<64, 32, 8, true, true>(J, pk, counter, sms, st) : run_gemm<64, 16, 8, true, true>(J, pk, counter, sms, st);
    else e = J.KC == 32 ? run_gemm<64, 32, 8, true>(J, pk, counter, sms, st) : run_gemm<64, 16, 8, true>(J, pk, counter, sms, st);
  } else {  // J2: U^T U, plain products
    if (J.BN == 128) e = J.KC == 32 ? run_gemm<128, 32, 8, false>(J, pk, counter, sms, st) : run_gemm<128, 16, 8, false>(J, pk, counter, sms, st);
    else if (J.BN == 96) e = J.KC == 32 ? run_gemm<96, 32, 8, false>(J, pk, counter, sms, st) : run_gemm<96, 16, 8, false>(J, pk, counter, sms, st);
    else e = J.KC == 32 ? run_gemm<64, 32, 8, false>(J, pk, counter, sms, st) : run_gemm<64, 16, 8, false>(J, pk, counter, sms, st);
  }
  return e;
}

// fixed-order sum of the job's split (x slab) partials
static cudaError_t reduce_job(const GemmJob& J, cudaStream_t st) {
  const int64_t n = J.split_stride;
  const int S = J.splits * J.nslab;
  if (S >= 4 * kRedGroups && n % 2 == 0 && n < (int64_t)148 * 8 * 512) {  // many splits of a small output
    k_reduce_splits_wide<<<(unsigned)((n / 2 + 31) / 32), 256, 0, st>>>(J.Cred, J.Cpart, n, S, J.split_stride);
    count_launch();
    return cudaGetLastError();
  }
  const int blocks = (int)std::min<int64_t>((n / 2 + 255) / 256, 148 * 8);
  k_reduce_splits<<<blocks, 256, 0, st>>>(J.Cred, J.Cpart, n, J.splits * J.nslab, J.split_stride);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t run_job(const GemmJob& J, const Packed& pk, unsigned* counter, int sms, cudaStream_t st,
                           cudaEvent_t after_gemm = nullptr) {
  cudaError_t e = run_gemm_only(J, pk, counter, sms, st);
  if (e != cudaSuccess) return e;
  if (after_gemm) cudaEventRecord(after_gemm, st);
  return reduce_job(J, st);
}

static void launch_frag(const GemmJob& J, const Packed& pk, bool a_side, cudaStream_t st, bool both = false,
                        const GemmJob* tailB = nullptr, int slab = 0) {
  FragArgs F;
  F.desc2 = nullptr;
  F.out2 = nullptr;
  F.tiles2 = 0;
  F.BT2 = 16;
  F.desc3 = tailB ? tailB->dB : nullptr;  // a tail job's B from the same staged rows
  F.out3 = tailB ? tailB->bfrag : nullptr;
  F.tiles3 = tailB ? tailB->tilesN : 0;
  F.BT3 = tailB ? tailB->BN : 16;
  if (both) {  // A (a_side ignored) and B of the same job from one staging of the rows
    a_side = true;
    F.desc2 = J.dB;
    F.out2 = J.bfrag;
    F.tiles2 = J.tilesN;
    F.BT2 = J.BN;
  }
  F.desc = a_side ? J.dA : J.dB;
  F.out = a_side ? J.afrag : J.bfrag;
  F.tiles = a_side ? J.tilesM : J.tilesN;
  F.BT = a_side ? J.BM : J.BN;
  F.KC = J.KC;
  F.nchunks = J.slab_chunks;  // buffer stride; this launch covers slab `slab`
  F.c_base = (int64_t)slab * J.slab_chunks;
  const int64_t count = std::min<int64_t>(J.slab_chunks, J.nchunks - F.c_base);
  F.nseg = J.dnseg;
  int off = 0;
  for (int sg = 0; sg < J.dnseg; ++sg) {
    const int id = J.dseg_id[sg];
    F.seg_ptr[sg] = id == 0 ? pk.Pr : (id == 1 ? pk.Xp : pk.Zp);
    F.seg_ld[sg] = id == 0 ? pk.ldP : (id == 1 ? pk.ldX : pk.ldZ);
    F.seg_off[sg] = off;
    off += J.KC * F.seg_ld[sg];
  }
  static uint64_t attr_mask = 0;
  set_once_per_device(attr_mask, [] {
    return cudaFuncSetAttribute(k_frag, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFragSmemMax);
  });
  F.nh = frag_nh((size_t)off);  // > 0: the plan materialises only operands whose stage fits
  k_frag<<<(unsigned)(F.nh * count), 256, (size_t)off / F.nh * sizeof(double), st>>>(F);
  count_launch();
}

cudaError_t launch_hessian(HessPlan* hp, const Dims& D, const Packed& pk, const double* Y, double* out,
                           int ld_out, double sign, cudaStream_t st) {
  cudaEventRecord(hp->ev[7], st);
  if (hp->small) {  // one launch; its time is reported as the J1 phase
    cudaEventRecord(hp->ev[0], st);
    SmallArgs A;
    A.N = D.N; A.K = D.K; A.q = D.q; A.d = D.d; A.f = D.f; A.n_p = D.n_p;
    A.n_beta = D.n_beta; A.off_gamma = D.off_gamma;
    A.Pr = pk.Pr; A.ldP = pk.ldP; A.Xp = pk.Xp; A.ldX = pk.ldX; A.Zp = pk.Zp; A.ldZ = pk.ldZ; A.Y = Y;
    A.part = hp->small_part; A.counter = hp->counters;
    A.out = out; A.ld_out = ld_out; A.sign = sign;
    k_hess_small<<<hp->small_grid, 256, 0, st>>>(A);
    count_launch();
    for (int i = 1; i <= 6; ++i) cudaEventRecord(hp->ev[i], st);
    return cudaGetLastError();
  }
  {  // operand materialisation: weights every evaluation, design-only products after a re-pack
    const GemmJob* jobs[4] = {&hp->j1, hp->has_j1b ? &hp->j1b : nullptr, hp->has_j2 ? &hp->j2 : nullptr,
                              hp->has_j2b ? &hp->j2b : nullptr};
    for (const GemmJob* J : jobs) {
      if (!J) continue;
      if (J->nslab > 1) continue;  // N-slabbed J1: materialised slab by slab below
      if (J->mat_a && J->mat_b && J->own_afrag && !J->b_design) {  // J2: A, B (+ the tail's B), one pass
        launch_frag(*J, pk, true, st, true, (J == &hp->j2 && hp->has_j2b) ? &hp->j2b : nullptr);
        continue;
      }
      if (J == &hp->j2b) continue;  // materialised with j2
      if (J->mat_b && (!J->b_design || !hp->bvalid)) launch_frag(*J, pk, false, st);
      if (J->mat_a && J->own_afrag) launch_frag(*J, pk, true, st);
    }
    hp->bvalid = true;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  cudaEventRecord(hp->ev[0], st);
  cudaError_t e = cudaSuccess;
  if (hp->j1.nslab > 1) {
    // N-slabs: per slab, both operands (and the tail's B) materialised from one staging of the
    // rows, then the main and tail GEMMs over that slab; the slab partials are reduced at the end
    // (the operand time is then counted in the GEMM phases)
    for (int sl = 0; sl < hp->j1.nslab && e == cudaSuccess; ++sl) {
      launch_frag(hp->j1, pk, true, st, true, hp->has_j1b ? &hp->j1b : nullptr, sl);
      e = run_gemm_only(hp->j1, pk, hp->counters, hp->sms, st, sl);
      if (e == cudaSuccess && hp->has_j1b) e = run_gemm_only(hp->j1b, pk, hp->counters, hp->sms, st, sl);
    }
    if (e != cudaSuccess) return e;
    cudaEventRecord(hp->ev[1], st);
    if ((e = reduce_job(hp->j1, st)) != cudaSuccess) return e;
    cudaEventRecord(hp->ev[2], st);
    cudaEventRecord(hp->ev[3], st);
    if (hp->has_j1b && (e = reduce_job(hp->j1b, st)) != cudaSuccess) return e;
  } else {
    e = run_job(hp->j1, pk, hp->counters, hp->sms, st, hp->ev[1]);
    if (e != cudaSuccess) return e;
    cudaEventRecord(hp->ev[2], st);
    if (hp->has_j1b) {
      e = run_job(hp->j1b, pk, hp->counters, hp->sms, st, hp->ev[3]);
      if (e != cudaSuccess) return e;
    } else {
      cudaEventRecord(hp->ev[3], st);
    }
  }
  cudaEventRecord(hp->ev[4], st);
  if (hp->has_j2) {
    e = run_job(hp->j2, pk, hp->counters + 1, hp->sms, st);
    if (e != cudaSuccess) return e;
    if (hp->has_j2b) {
      e = run_job(hp->j2b, pk, hp->counters + 1, hp->sms, st);
      if (e != cudaSuccess) return e;
    }
    const int E = D.q + D.d + D.f, F = D.d + D.f;
    {
      const int items = (D.K + 7) / 8 * hp->ar_ep * hp->ar_fp * hp->ar_splits;
      const int64_t tstride = ((int64_t)D.K * E * F + 1) / 2 * 2;
#define MNL_ARROW(MT_, NT_)                                                                                  \
  do {                                                                                                       \
    static uint64_t attr_mask_ = 0;                                                                          \
    set_once_per_device(attr_mask_, [] {                                                                     \
      return cudaFuncSetAttribute(k_arrow<MT_, NT_>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024); \
    });                                                                                                      \
    k_arrow<MT_, NT_><<<items, 256, (size_t)2 * hp->ar_ci * hp->ar_rs * sizeof(double), st>>>(               \
        D.N, D.K, D.q, D.d, D.f, hp->ar_splits, pk.Npad, hp->ar_ep, hp->ar_fp, hp->ar_ci, hp->ar_rs, pk.Pr,   \
        pk.ldP, pk.Xp, pk.ldX, pk.Zp, pk.ldZ, Y, hp->Tpart, tstride);                                        \
  } while (0)
      if (hp->ar_mt == 8 && hp->ar_nt == 4) MNL_ARROW(8, 4);
      else if (hp->ar_mt == 8) MNL_ARROW(8, 2);
      else if (hp->ar_mt == 6 && hp->ar_nt == 4) MNL_ARROW(6, 4);
      else if (hp->ar_mt == 6) MNL_ARROW(6, 2);
      else if (hp->ar_mt == 4 && hp->ar_nt == 4) MNL_ARROW(4, 4);
      else if (hp->ar_mt == 4) MNL_ARROW(4, 2);
      else if (hp->ar_nt == 4) MNL_ARROW(2, 4);
      else MNL_ARROW(2, 2);
#undef MNL_ARROW
      count_launch();
    }
    const int64_t n = (int64_t)D.K * E * F;
    if (hp->ar_splits >= 4 * kRedGroups && n % 2 == 0)
      k_reduce_splits_wide<<<(unsigned)((n / 2 + 31) / 32), 256, 0, st>>>(hp->T, hp->Tpart, n, hp->ar_splits, n);
    else
      k_reduce_splits<<<(int)std::min<int64_t>((n / 2 + 256) / 256, 1024), 256, 0, st>>>(hp->T, hp->Tpart, n,
                                                                                         hp->ar_splits, (n + 1) / 2 * 2);
    count_launch();
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  cudaEventRecord(hp->ev[5], st);
  AsmArgs A;
  A.K = D.K; A.q = D.q; A.d = D.d; A.f = D.f;
  A.n_beta = D.n_beta; A.off_gamma = D.off_gamma; A.n_p = D.n_p;
  A.C1 = hp->j1.Cred; A.ld1 = hp->j1.ldc;
  A.C1b = hp->has_j1b ? hp->j1b.Cred : nullptr; A.ld1b = hp->has_j1b ? hp->j1b.ldc : 0; A.n1a = hp->n1a;
  A.C2 = hp->has_j2 ? hp->j2.Cred : nullptr; A.ld2 = hp->has_j2 ? hp->j2.ldc : 0;
  A.C2b = hp->has_j2b ? hp->j2b.Cred : nullptr; A.ld2b = hp->has_j2b ? hp->j2b.ldc : 0;
  A.n2a = hp->has_j2b ? hp->n2a : (1 << 30);
  A.T = hp->T;
  A.out = out; A.ld_out = ld_out; A.sign = sign;
  const int64_t total = (int64_t)D.n_p * D.n_p;
  const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 16);
  k_assemble<<<blocks, 256, 0, st>>>(A);
  count_launch();
  cudaEventRecord(hp->ev[6], st);
  return cudaGetLastError();
}

void hess_plan_design_changed(HessPlan* hp) {
  if (hp) hp->bvalid = false;
}

void hess_last_times(HessPlan* hp, double out[7]) {
  // [0] J1 GEMM (128-column tiles), [1] its split reduction, [2] J1 tail GEMM (narrow tile),
  // [3] its reduction, [4] Z/Y blocks (J2 + same-alternative), [5] assembly,
  // [6] operand materialisation before J1 (k_frag: weights every evaluation, design-only products
  //     once per packed design)
  for (int i = 0; i < 7; ++i) {
    float ms = 0.f;
    if (!hp) { out[i] = 0.0; continue; }
    cudaEvent_t a = i < 6 ? hp->ev[i] : hp->ev[7], b = i < 6 ? hp->ev[i + 1] : hp->ev[0];
    if (cudaEventElapsedTime(&ms, a, b) != cudaSuccess) ms = 0.f;
    out[i] = ms;
  }
}

// ---- packed upper triangle (the data-parallel exchange) -----------------------
// Row i of the upper triangle (columns i..n-1) starts at off(i) = i n - i (i - 1) / 2. One CTA per
// row; pack reads H[i][i..] and writes contiguously (coalesced both sides); unpack writes the
// row and mirrors it into column i (exactly symmetric result).
__global__ void k_sym_pack(int n, const double* __restrict__ H, double* __restrict__ out) {
  const int64_t i = blockIdx.x;
  const int64_t off = i * n - i * (i - 1) / 2;
  for (int64_t j = i + threadIdx.x; j < n; j += blockDim.x) out[off + (j - i)] = H[i * n + j];
}
__global__ void k_sym_unpack(int n, const double* __restrict__ in, double* __restrict__ H) {
  const int64_t i = blockIdx.x;
  const int64_t off = i * n - i * (i - 1) / 2;
  for (int64_t j = i + threadIdx.x; j < n; j += blockDim.x) {
    const double v = in[off + (j - i)];
    H[i * n + j] = v;
    H[j * n + i] = v;
  }
}

cudaError_t launch_sym_pack(int n, const double* H, double* out, cudaStream_t st) {
  k_sym_pack<<<n, 256, 0, st>>>(n, H, out);
  count_launch();
  return cudaGetLastError();
}
cudaError_t launch_sym_unpack(int n, const double* in, double* H, cudaStream_t st) {
  k_sym_unpack<<<n, 256, 0, st>>>(n, in, H);
  count_launch();
  return cudaGetLastError();
}

}  // namespace mnl
