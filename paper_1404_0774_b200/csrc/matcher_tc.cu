// matcher_tc.cu — K2, the tcgen05 range x (domain, isometry) matcher for n in {2, 4, 8}.
//
// The dense part of Searcher::search_impl (proj/src/encoder.cpp:236-241) is the
// correlation acc = sum_i q[perm_s(i)] * b_i for every (range, domain, isometry).  Here
// it is one GEMM per CTA tile:   D[128 ranges, 256 columns] = A[128, K] * B[256, K]^T
// with A = range pixels b (fp16, exact) and B = the pool's 32 domains x 8 isometries
// of 2x2 group sums q (fp16, exact, q <= 1020).  Every product is an integer < 2^18 and
// every partial sum an integer < 64*1020*255 < 2^24, so the fp32 TMEM accumulators are
// EXACT integers (the same bits the reference's int accumulators hold).
//
// CTA = (128-range M tile, contiguous chunk of 256-column domain tiles); 12 warps:
//   warp 0      bulk-copy producer: pool tiles (contiguous 32*K*16 B) -> smem ring
//   warp 1      MMA issuer: one elected thread issues K/16 tcgen05.mma per tile
//   warp 2      TMEM allocator (512 columns = two 256-column accumulators)
//   warps 4-7   epilogue group 0 (even tiles, accumulator 0)
//   warps 8-11  epilogue group 1 (odd tiles, accumulator 1)
// Each epilogue thread owns one TMEM lane = one range: it loads 32 columns (4 domains)
// at a time with tcgen05.ld, applies the 8-isometry group bound (an integer max/min
// over the 8 correlations against the least-squares pruning interval), and sends the
// rare survivors through the reference-exact fp64 evaluation (common.cuh).  The
// R x D x 8 error matrix never leaves the SM.
#include "common.cuh"
#include "tc_ptx.cuh"

namespace ficb {

constexpr int kTcThreads = 384;
constexpr int kTcStages = 4;
constexpr int kTileCols = kDomainsPerTile * kSyms;  // 256
constexpr uint32_t kTmemCols = 512;

// Per-epilogue-warp survivor queue: domain groups whose 8-isometry bound did not prune
// them, with their 8 correlations, processed 32 at a time (one per lane) so the fp64
// reference evaluation runs with the whole warp busy instead of one lane at a time.
struct QEntry {
  int d;
  int owner;            // lane (= range) the group belongs to
  uint32_t acc[kSyms];  // fp32 bits of the exact correlations
  int pad[2];
};
constexpr int kQCap = 64;
constexpr int kEpiWarps = 8;

struct TcSmemLayout {
  uint32_t a_bytes, b_bytes, a_off, b_off, bar_off, best_off, q_off, meta_off, total;
};

__host__ __device__ inline TcSmemLayout tc_smem_layout(int K) {
  TcSmemLayout L;
  L.a_bytes = kRangesPerTile * K * 2;
  L.b_bytes = kDomainsPerTile * K * 16;
  L.a_off = 0;
  L.b_off = (L.a_bytes + 1023) & ~1023u;
  L.bar_off = L.b_off + kTcStages * L.b_bytes;
  L.best_off = L.bar_off + 256;
  L.q_off = L.best_off;
  L.meta_off = L.q_off + kEpiWarps * kQCap * sizeof(QEntry);
  L.total = L.meta_off + kEpiWarps * kDomainsPerTile * sizeof(DomainMetaF) + 1024;  // + alignment slack
  return L;
}


// Evaluates the queued groups 32 at a time (lane i takes entry base+i, whatever range it
// belongs to: the owner's state is fetched with shuffles), then merges the results into
// the owners in queue order.  Per owner, entries are queued in increasing domain order
// and each entry's isometries are tried in order, so strict-< updates reproduce the
// reference's first-minimum tie-breaking.
template <int NN>
__device__ __noinline__ void flush_queue(QEntry* queue, int qcount, RangeState& st, const Geometry& g,
                                         const DomainMetaF* __restrict__ meta_f,
                                         const DomainMetaI* __restrict__ meta_i,
                                         const unsigned char* __restrict__ pool,
                                         const unsigned char* __restrict__ img, unsigned long long* gbest,
                                         unsigned long long* counters, int lane) {
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  __syncwarp();
  for (int base = 0; base < qcount; base += 32) {
    const int i = base + lane;
    const bool valid = i < qcount;
    QEntry e;
    if (valid) e = queue[i];
    const int owner = valid ? e.owner : lane;
    const double o_ssb = __shfl_sync(0xffffffffu, st.ssb, owner);
    const double o_thr = __shfl_sync(0xffffffffu, st.thr, owner);
    const int o_sb = __shfl_sync(0xffffffffu, st.sb, owner);
    const float o_sqrtT = __shfl_sync(0xffffffffu, st.sqrtT, owner);
    const int o_x0 = __shfl_sync(0xffffffffu, st.x0, owner);
    const int o_y0 = __shfl_sync(0xffffffffu, st.y0, owner);
    double R = inf;
    int rs = 0;
    unsigned rqs = 0, rqo = 0;
    if (valid) {
      count(counters, 1, g);
      const DomainMetaI mi = meta_i[e.d];
      if (mi.den >= 0) {
        const DomainMetaF mf = meta_f[e.d];
        uint32_t bpk[NN / 4];
        load_range_packed<NN>(img, g, o_x0, o_y0, bpk);
        const float center = mf.a * (float)o_sb;
        const float rad = __fmaf_rn(mf.e, o_sqrtT, -kBoundSlack);
        double thr = o_thr;
        for (int s = 0; s < kSyms; ++s) {
          const float av = __uint_as_float(e.acc[s]);
          if (!(g.flags & 1) && (av - center <= rad) && (center - av <= rad)) continue;  // per-isometry bound
          unsigned qs = 0, qo = 0;
          const double rv = eval_candidate<NN>(g, e.d, s, (long long)av, mi, o_sb, o_ssb, thr, bpk, pool, img,
                                               o_x0, o_y0, qs, qo, counters);
          if (rv < R) {
            R = rv;
            rs = s;
            rqs = qs;
            rqo = qo;
            if (rv < thr) thr = rv;
          }
        }
      }
    }
    // merge into the owners, in queue order
    uint32_t found = __ballot_sync(0xffffffffu, R < inf);
    while (found) {
      const int k = __ffs(found) - 1;
      found &= found - 1;
      const double Rk = __shfl_sync(0xffffffffu, R, k);
      const int ok = __shfl_sync(0xffffffffu, owner, k);
      const int dk = __shfl_sync(0xffffffffu, valid ? e.d : 0, k);
      const int sk = __shfl_sync(0xffffffffu, rs, k);
      const unsigned qsk = __shfl_sync(0xffffffffu, rqs, k);
      const unsigned qok = __shfl_sync(0xffffffffu, rqo, k);
      if (lane == ok && Rk < st.best) {
        st.best = Rk;
        st.bd = dk;
        st.bs = sk;
        st.bqs = qsk;
        st.bqo = qok;
      }
    }
    if (st.best < st.thr) {
      st.thr = st.best;
      st.sqrtT = prune_sqrtT(st.ssb, st.thr, NN);
      publish_best(gbest, st.r, st.best);
    }
  }
  __syncwarp();
}

template <int NN>
__global__ void __launch_bounds__(kTcThreads, 1)
matcher_tc_kernel(const unsigned char* __restrict__ img, Geometry g, const unsigned char* __restrict__ pool,
                  const DomainMetaF* __restrict__ meta_f, const DomainMetaI* __restrict__ meta_i,
                  const RangeMeta* __restrict__ rmeta, int tiles_per_chunk, int n_tiles,
                  Partial* __restrict__ partials, unsigned long long* __restrict__ gbest,
                  unsigned long long* __restrict__ counters) {
  constexpr int K = NN < 16 ? 16 : NN;
  extern __shared__ unsigned char smem_raw[];
  unsigned char* smem = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const TcSmemLayout L = tc_smem_layout(K);
  unsigned char* sA = smem + L.a_off;
  unsigned char* sB = smem + L.b_off;
  uint64_t* full_bar = reinterpret_cast<uint64_t*>(smem + L.bar_off);
  uint64_t* empty_bar = full_bar + kTcStages;
  uint64_t* tfull_bar = empty_bar + kTcStages;
  uint64_t* tempty_bar = tfull_bar + 2;
  uint32_t* tmem_base_smem = reinterpret_cast<uint32_t*>(tempty_bar + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m_tile = blockIdx.x;
  const int t_begin = blockIdx.y * tiles_per_chunk;
  const int t_end = min(n_tiles, t_begin + tiles_per_chunk);
  const int ntiles = max(0, t_end - t_begin);

  // ---- setup: barriers, TMEM, A operand (range pixels) ----
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], 4);  // one elected lane per epilogue warp
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<kTmemCols>(tmem_base_smem);
  if (threadIdx.x < kRangesPerTile) {
    // A row = range pixels in row-major order, fp16, K-major no-swizzle core matrices:
    // offset(row, k) = (row/8)*K*16 + (k/8)*128 + (row%8)*16 + (k%8)*2
    const int row = threadIdx.x;
    const int r = m_tile * kRangesPerTile + row;
    const bool valid = r < g.R;
    int x0 = 0, y0 = 0;
    if (valid) range_origin(g, r, x0, y0);
#pragma unroll
    for (int kc = 0; kc < K / 8; ++kc) {
      uint32_t w[4];
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        uint32_t h2 = 0;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int k = kc * 8 + 2 * t + u;
          unsigned short hv = 0;
          if (valid && k < g.N)
            hv = __half_as_ushort(__ushort2half_rn(img[(long long)(y0 + k / g.n) * g.W + x0 + k % g.n]));
          h2 |= (uint32_t)hv << (16 * u);
        }
        w[t] = h2;
      }
      *reinterpret_cast<uint4*>(sA + (row >> 3) * K * 16 + kc * 128 + (row & 7) * 16) =
          make_uint4(w[0], w[1], w[2], w[3]);
    }
  }
  ptx::fence_proxy_async_smem();  // generic-proxy writes of A -> visible to the tensor core
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = *tmem_base_smem;

  if (warp == 0) {
    // ================= producer =================
    if (lane == 0) {
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kTcStages;
        const uint32_t ph = (i / kTcStages) & 1;
        ptx::mbar_wait(&empty_bar[s], ph ^ 1);
        ptx::mbar_arrive_expect_tx(&full_bar[s], L.b_bytes);
        ptx::bulk_g2s(sB + s * L.b_bytes, pool + (long long)(t_begin + i) * L.b_bytes, L.b_bytes, &full_bar[s]);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_f16_f32(kRangesPerTile, kTileCols);
      const uint32_t a_base = ptx::smem_addr(sA);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kTcStages;
        const uint32_t ph = (i / kTcStages) & 1;
        const int buf = i & 1;
        const uint32_t bph = (i >> 1) & 1;
        ptx::mbar_wait(&tempty_bar[buf], bph ^ 1);
        ptx::mbar_wait(&full_bar[s], ph);
        ptx::tc_fence_after();
        const uint32_t b_base = ptx::smem_addr(sB + s * L.b_bytes);
#pragma unroll
        for (int kk = 0; kk < K / 16; ++kk) {
          const uint64_t ad = ptx::smem_desc(a_base + kk * 256, 128, K * 16);
          const uint64_t bd = ptx::smem_desc(b_base + kk * 256, 128, K * 16);
          ptx::mma_f16_ss(tmem_base + buf * kTileCols, ad, bd, idesc, kk > 0 ? 1u : 0u);
        }
        ptx::tc_commit(&empty_bar[s]);   // smem stage free once these MMAs have read it
        ptx::tc_commit(&tfull_bar[buf]); // accumulator ready for the epilogue
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue =================
    const int wg = (warp - 4) >> 2;          // 0 or 1: which accumulator / tile parity
    const int quarter = warp & 3;            // TMEM lane quarter this warp may access
    const int row = quarter * 32 + lane;
    const int r = m_tile * kRangesPerTile + row;
    QEntry* queue = reinterpret_cast<QEntry*>(smem + L.q_off) + (warp - 4) * kQCap;
    DomainMetaF* smeta = reinterpret_cast<DomainMetaF*>(smem + L.meta_off) + (warp - 4) * kDomainsPerTile;
    RangeState st;
    st.r = r;
    st.best = st.thr = __longlong_as_double(0x7ff0000000000000ll);
    st.bd = -1;
    st.bs = 0;
    st.bqs = st.bqo = 0;
    st.active = false;
    st.sb = 0;
    st.ssb = 0.0;
    st.x0 = st.y0 = 0;
    if (r < g.R) {
      const RangeMeta m = rmeta[r];
      range_origin(g, r, st.x0, st.y0);
      st.sb = m.sb;
      st.ssb = (double)m.var / (double)g.N;
      st.active = !m.shadow;
    }
    st.sqrtT = st.active ? -1e30f : 1e30f;  // inactive lanes prune everything
    const float sb_f = (float)st.sb;
    const uint32_t lane_addr = (uint32_t)(quarter * 32) << 16;
    int qcount = 0;  // warp-uniform

    for (int i = wg; i < ntiles; i += 2) {
      const uint32_t bph = (i >> 1) & 1;
      const int d0 = (t_begin + i) * kDomainsPerTile;
      __syncwarp();
      smeta[lane] = meta_f[d0 + lane];
      refresh_thr(st, gbest, NN);
      __syncwarp();
      ptx::mbar_wait(&tfull_bar[wg], bph);
      ptx::tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < kTileCols / 64; ++h) {
        __syncwarp();  // tcgen05.ld is .sync.aligned
        uint32_t v[64];
        ptx::tmem_ld_32x32b_x32(tmem_base + lane_addr + wg * kTileCols + h * 64, v);
        ptx::tmem_ld_32x32b_x32(tmem_base + lane_addr + wg * kTileCols + h * 64 + 32, v + 32);
        ptx::tmem_ld_wait();
        // 8-isometry group bound for 8 domains, branch-free
        uint32_t gmask = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float* f = reinterpret_cast<const float*>(v + 8 * j);
          const float mx = fmaxf(fmaxf(fmaxf(f[0], f[1]), fmaxf(f[2], f[3])), fmaxf(fmaxf(f[4], f[5]), fmaxf(f[6], f[7])));
          const float mn = fminf(fminf(fminf(f[0], f[1]), fminf(f[2], f[3])), fminf(fminf(f[4], f[5]), fminf(f[6], f[7])));
          const DomainMetaF m = smeta[h * 8 + j];
          const float center = m.a * sb_f;
          const float rad = __fmaf_rn(m.e, st.sqrtT, -kBoundSlack);
          const bool keep = (mx - center > rad) | (center - mn > rad);
          gmask |= (uint32_t)keep << j;
        }
        if (g.flags & 1) gmask = st.active ? 0xFFu : 0u;
        if (__any_sync(0xffffffffu, gmask != 0)) {
          // push surviving groups (domain-major, lane-minor) onto the warp's queue
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const bool mine = (gmask >> j) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, mine);
            if (bal == 0) continue;
            const int cnt = __popc(bal);
            if (qcount + cnt > kQCap) {
              flush_queue<NN>(queue, qcount, st, g, meta_f, meta_i, pool, img, gbest, counters, lane);
              qcount = 0;
            }
            if (mine) {
              QEntry* e = queue + qcount + __popc(bal & ((1u << lane) - 1u));
              e->d = d0 + h * 8 + j;
              e->owner = lane;
              *reinterpret_cast<uint4*>(e->acc) = make_uint4(v[8 * j], v[8 * j + 1], v[8 * j + 2], v[8 * j + 3]);
              *reinterpret_cast<uint4*>(e->acc + 4) = make_uint4(v[8 * j + 4], v[8 * j + 5], v[8 * j + 6], v[8 * j + 7]);
            }
            qcount += cnt;
          }
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&tempty_bar[wg]);  // accumulator free for the MMA
      if (qcount >= 32) {
        flush_queue<NN>(queue, qcount, st, g, meta_f, meta_i, pool, img, gbest, counters, lane);
        qcount = 0;
      }
    }
    if (qcount > 0) flush_queue<NN>(queue, qcount, st, g, meta_f, meta_i, pool, img, gbest, counters, lane);
    if (r < g.R)
      partials[(long long)(blockIdx.y * 2 + wg) * g.R + r] = Partial{st.best, st.bd, st.bs, st.bqs, st.bqo};
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tmem_base);
  }
}

size_t tc_smem_bytes(int K) {
  const TcSmemLayout L = tc_smem_layout(K);
  // at least ~116 KB so exactly one CTA (and one 512-column TMEM allocation) lives per SM
  return L.total < 118 * 1024 ? 118 * 1024 : L.total;
}

bool tc_supported(const Geometry& g) { return g.N == 4 || g.N == 16 || g.N == 64; }

template <int NN>
static cudaError_t launch_tc(const unsigned char* img, const Geometry& g, const unsigned char* pool,
                             const DomainMetaF* meta_f, const DomainMetaI* meta_i, const RangeMeta* rmeta,
                             int n_chunks, int tiles_per_chunk, Partial* partials, unsigned long long* gbest,
                             unsigned long long* counters, cudaStream_t st) {
  const int n_tiles = g.D_pad / kDomainsPerTile;
  dim3 grid((g.R + kRangesPerTile - 1) / kRangesPerTile, n_chunks);
  const size_t smem = tc_smem_bytes(g.K);
  const cudaError_t e =
      cudaFuncSetAttribute(matcher_tc_kernel<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  matcher_tc_kernel<NN><<<grid, kTcThreads, smem, st>>>(img, g, pool, meta_f, meta_i, rmeta, tiles_per_chunk,
                                                        n_tiles, partials, gbest, counters);
  return cudaGetLastError();
}

cudaError_t launch_matcher_tc(const unsigned char* img, const Geometry& g, const unsigned char* pool,
                              const DomainMetaF* meta_f, const DomainMetaI* meta_i, const RangeMeta* rmeta,
                              int n_chunks, int tiles_per_chunk, Partial* partials, unsigned long long* gbest,
                              unsigned long long* counters, cudaStream_t st) {
  if (g.N == 4)
    return launch_tc<4>(img, g, pool, meta_f, meta_i, rmeta, n_chunks, tiles_per_chunk, partials, gbest, counters, st);
  if (g.N == 16)
    return launch_tc<16>(img, g, pool, meta_f, meta_i, rmeta, n_chunks, tiles_per_chunk, partials, gbest, counters, st);
  return launch_tc<64>(img, g, pool, meta_f, meta_i, rmeta, n_chunks, tiles_per_chunk, partials, gbest, counters, st);
}

}  // namespace ficb
