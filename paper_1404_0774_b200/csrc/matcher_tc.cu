// matcher_tc.cu — K2, the tcgen05 range x (domain, isometry) matcher for n in {2, 4, 8}.
//
// The dense part of Searcher::search_impl (proj/src/encoder.cpp:236-241) is the
// correlation acc = sum_i q[perm_s(i)] * b_i for every (range, domain, isometry).  Here it
// is a GEMM per CTA tile:  D[256 ranges, 128 columns] = A[256, K] * B[128, K]^T  with
// A = range pixels b (fp16, exact) and B = the pool's 16 domains x 8 isometries of 2x2
// group sums q (fp16, exact, q <= 1020).  Every product is an integer < 2^18 and every
// partial sum an integer < 64*1020*255 < 2^24, so the fp32 TMEM accumulators hold EXACT
// integers (the same values the reference's int accumulators hold).
//
// CTA = 256 ranges (two 128-lane M sub-tiles sharing every B tile, which halves the L2
// traffic of streaming the pool) x a contiguous chunk of 16-domain tiles; 20 warps:
//   warp 0       bulk-copy producer: pool tiles (contiguous 16*K*16 B) -> smem ring
//   warp 1       MMA issuer: one thread issues 2 * K/16 tcgen05.mma (M=128, N=128) per tile
//   warp 2       TMEM allocator (512 columns = 2 sub-tiles x 2 buffers x 128 columns)
//   warps 4-19   epilogue: 4 groups of 4 warps, group (buffer b, sub-tile m) owns the
//                accumulator (2b+m) of every tile with parity b
// Each epilogue thread owns one TMEM lane = one range.  Per 64 columns (8 domains) it
// loads the accumulators with tcgen05.ld and applies the 8-isometry group bound (3-input
// min/max over the 8 exact correlations against the least-squares pruning interval); the
// rare groups that survive go to a per-warp queue in shared memory and are evaluated 32
// at a time (one per lane) by the reference-exact fp64 path.  The R x D x 8 error matrix
// never leaves the SM.
#include "common.cuh"
#include "tc_ptx.cuh"

namespace ficb {

constexpr int kTcThreads = 640;
constexpr int kTcStages = 6;
constexpr int kTcRows = 256;                          // ranges per CTA (two M sub-tiles)
constexpr int kTcTileDomains = 16;                    // domains per MMA tile
constexpr int kTileCols = kTcTileDomains * kSyms;     // 128 = MMA N
constexpr uint32_t kTmemCols = 512;
constexpr int kEpiWarps = 16;

// Survivor queue entry: a domain group whose 8-isometry bound did not prune it.
struct QEntry {
  int d;
  int owner;            // lane (= range row within the warp)
  float a, e;           // DomainMetaF of d
  uint32_t acc[kSyms];  // fp32 bits of the exact correlations
  long long sq, den;    // DomainMetaI of d
};
struct TileMeta {       // per-domain metadata of the tile being processed (smem copy)
  DomainMetaF f;
  DomainMetaI i;
};
constexpr int kQCap = 32;

// Mutable per-range state of one epilogue group, kept in shared memory so the rare
// survivor path (a non-inlined function) can update it without forcing the hot loop's
// registers onto the stack.
struct RowState {
  double best;  // best residual among this group's candidates
  double thr;   // pruning bar: min(best, any published residual)
  double ssb;   // range_var / N
  int bd, bs;
  unsigned qs, qo;
  int sb, x0, y0, r;
  float sqrtT;
  int active;
  int pad[2];
};

struct TcSmemLayout {
  uint32_t a_bytes, b_bytes, a_off, b_off, bar_off, q_off, rows_off, meta_off, total;
};

__host__ __device__ inline TcSmemLayout tc_smem_layout(int K) {
  TcSmemLayout L;
  L.a_bytes = kTcRows * K * 2;
  L.b_bytes = kTcTileDomains * K * 16;
  L.a_off = 0;
  L.b_off = (L.a_bytes + 1023) & ~1023u;
  L.bar_off = L.b_off + kTcStages * L.b_bytes;
  L.q_off = L.bar_off + 256;
  L.rows_off = L.q_off + kEpiWarps * kQCap * (uint32_t)sizeof(QEntry);
  L.meta_off = L.rows_off + 4 * 128 * (uint32_t)sizeof(RowState);
  L.total = L.meta_off + kEpiWarps * kTcTileDomains * (uint32_t)sizeof(TileMeta);
  return L;
}

// Evaluates the queued groups 32 at a time (lane i takes entry base+i, whichever range
// it belongs to) and merges the results into the owners' RowState in queue order.  Per
// owner, entries are queued in increasing domain order and each entry's isometries are
// tried in order, so strict-< updates reproduce the reference's first-minimum tie-break.
template <int NN>
__device__ __noinline__ void flush_queue(const QEntry* queue, int qcount, RowState* rows, const Geometry& g,
                                         const DomainMetaF* __restrict__ meta_f,
                                         const DomainMetaI* __restrict__ meta_i,
                                         const unsigned char* __restrict__ pool,
                                         const unsigned char* __restrict__ img, unsigned long long* gbest,
                                         unsigned long long* counters) {
  const int lane = threadIdx.x & 31;
  const double inf = __longlong_as_double(0x7ff0000000000000ll);
  __syncwarp();
  for (int base = 0; base < qcount; base += 32) {
    const int i = base + lane;
    const bool valid = i < qcount;
    int d = 0, owner = 0;
    double R = inf;
    int rs = 0;
    unsigned rqs = 0, rqo = 0;
    if (valid) {
      const QEntry e = queue[i];
      d = e.d;
      owner = e.owner;
      count(counters, 1, g);
      const DomainMetaI mi{e.sq, e.den};
      const RowState& row = rows[owner];
      if (mi.den >= 0) {
        const float center = e.a * (float)row.sb;
        const float rad = __fmaf_rn(e.e, row.sqrtT, -kBoundSlack);
        double thr = row.thr;
#pragma unroll 1
        for (int s = 0; s < kSyms; ++s) {
          const float av = __uint_as_float(e.acc[s]);
          if (!(g.flags & 1) && (av - center <= rad) && (center - av <= rad)) continue;  // per-isometry bound
          unsigned qs = 0, qo = 0;
          const double rv = eval_candidate<NN>(g, d, s, (long long)av, mi, row.sb, row.ssb, thr, nullptr, pool, img,
                                               row.x0, row.y0, qs, qo, counters);
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
    // merge into the owners, in queue order (one entry at a time: same-owner entries
    // in this round must be applied in order)
    uint32_t found = __ballot_sync(0xffffffffu, R < inf);
    while (found) {
      const int k = __ffs(found) - 1;
      found &= found - 1;
      if (lane == k) {
        RowState& row = rows[owner];
        // lexicographic (R, domain, isometry): independent of the order tiles were scanned in
        if (R < row.best || (R == row.best && (d < row.bd || (d == row.bd && rs < row.bs)))) {
          row.best = R;
          row.bd = d;
          row.bs = rs;
          row.qs = rqs;
          row.qo = rqo;
          if (R < row.thr) {
            row.thr = R;
            row.sqrtT = prune_sqrtT(row.ssb, R, NN);
            publish_best(gbest, row.r, R);
          }
        }
      }
      __syncwarp();
    }
  }
  __syncwarp();
}

template <int NN>
__global__ void __launch_bounds__(kTcThreads, 1)
matcher_tc_kernel(const unsigned char* __restrict__ img, Geometry g, const unsigned char* __restrict__ pool,
                  const DomainMetaF* __restrict__ meta_f, const DomainMetaI* __restrict__ meta_i,
                  const RangeMeta* __restrict__ rmeta, int tiles_per_chunk, int n_tiles, int tile_step,
                  Partial* __restrict__ partials, unsigned long long* __restrict__ gbest,
                  unsigned long long* __restrict__ counters) {
  constexpr int K = NN < 16 ? 16 : NN;
  // chunks split a (possibly strided) sequence of tiles: local tile i is physical tile
  // (t_begin + i) * tile_step; tile_step > 1 is the sparse pre-pass that seeds the bar
  auto phys_raw = [tile_step](int v) { return v * tile_step; };
  // The no-swizzle operand layout and the 16-byte bulk copies need only 128-byte
  // alignment; indexing the extern array directly keeps accesses in the shared window.
  extern __shared__ __align__(1024) unsigned char smem[];
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
  // CTAs of one wave (different M tiles, same chunk) start the chunk at staggered tiles so
  // they do not all request the same pool lines from L2 at the same moment; the result does
  // not depend on the order (survivor merges are lexicographic in (R, domain, isometry)).
  const int rot = (ntiles > 0 && (g.flags & 64) == 0) ? (int)(((long long)m_tile * 2654435761ll) % ntiles) : 0;
  auto phys = [=](int v) {
    const int k = v - t_begin;
    const int kk = k + rot >= ntiles ? k + rot - ntiles : k + rot;
    return phys_raw(t_begin + kk);
  };

  // ---- setup: barriers, TMEM, A operand (range pixels) ----
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < kTcStages; ++s) {
      ptx::mbar_init(&full_bar[s], 1);
      ptx::mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      ptx::mbar_init(&tfull_bar[b], 1);
      ptx::mbar_init(&tempty_bar[b], 8);  // one elected lane per epilogue warp of both sub-tiles
    }
    ptx::fence_mbar_init();
  }
  if (warp == 2) ptx::tmem_alloc<kTmemCols>(tmem_base_smem);
  if (threadIdx.x < kTcRows) {
    // A row = range pixels in row-major order, fp16, K-major no-swizzle core matrices:
    // offset(row, k) = (row/8)*K*16 + (k/8)*128 + (row%8)*16 + (k%8)*2
    const int row = threadIdx.x;
    const int r = m_tile * kTcRows + row;
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
          if (valid && k < NN)
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
        if ((g.flags & 32) && counters && blockIdx.x == 0 && blockIdx.y == 0 && i < 64) counters[8 + i] = clock64();
        ptx::mbar_arrive_expect_tx(&full_bar[s], L.b_bytes);
        ptx::bulk_g2s(sB + s * L.b_bytes, pool + (long long)phys(t_begin + i) * L.b_bytes, L.b_bytes, &full_bar[s]);
      }
    }
  } else if (warp == 1) {
    // ================= MMA issuer =================
    if (lane == 0) {
      constexpr uint32_t idesc = ptx::idesc_f16_f32(128, kTileCols);
      const uint32_t a_base = ptx::smem_addr(sA);
      for (int i = 0; i < ntiles; ++i) {
        const int s = i % kTcStages;
        const uint32_t ph = (i / kTcStages) & 1;
        const int buf = i & 1;
        const uint32_t bph = (i >> 1) & 1;
        ptx::mbar_wait(&tempty_bar[buf], bph ^ 1);
        ptx::mbar_wait(&full_bar[s], ph);
        ptx::tc_fence_after();
        if ((g.flags & 32) && counters && blockIdx.x == 0 && blockIdx.y == 0 && i < 64) counters[8 + 64 + i] = clock64();
        const uint32_t b_base = ptx::smem_addr(sB + s * L.b_bytes);
        if (!(g.flags & 16)) {  // debug: flags&16 skips the MMAs
#pragma unroll
          for (int m = 0; m < 2; ++m) {
#pragma unroll
            for (int kk = 0; kk < K / 16; ++kk) {
              const uint64_t ad = ptx::smem_desc(a_base + m * 128 * K * 2 + kk * 256, 128, K * 16);
              const uint64_t bd = ptx::smem_desc(b_base + kk * 256, 128, K * 16);
              ptx::mma_f16_ss(tmem_base + (buf * 2 + m) * kTileCols, ad, bd, idesc, kk > 0 ? 1u : 0u);
            }
          }
        }
        ptx::tc_commit(&empty_bar[s]);   // smem stage free once these MMAs have read it
        ptx::tc_commit(&tfull_bar[buf]); // accumulators ready for the epilogue
      }
    }
  } else if (warp >= 4) {
    // ================= epilogue =================
    const int e = warp - 4;             // 0..15
    const int grp = e >> 2;             // 0..3
    const int buf = grp >> 1;           // tile parity handled
    const int sub = grp & 1;            // M sub-tile
    const int quarter = warp & 3;       // TMEM lane quarter this warp may access
    const int row = sub * 128 + quarter * 32 + lane;
    const int r = m_tile * kTcRows + row;
    QEntry* queue = reinterpret_cast<QEntry*>(smem + L.q_off) + e * kQCap;
    RowState* rows = reinterpret_cast<RowState*>(smem + L.rows_off) + grp * 128 + quarter * 32;
    TileMeta* smeta = reinterpret_cast<TileMeta*>(smem + L.meta_off) + e * kTcTileDomains;
    {
      RowState rs;
      rs.best = rs.thr = __longlong_as_double(0x7ff0000000000000ll);
      rs.bd = -1;
      rs.bs = 0;
      rs.qs = rs.qo = 0;
      rs.active = 0;
      rs.sb = 0;
      rs.ssb = 0.0;
      rs.x0 = rs.y0 = 0;
      rs.r = r;
      if (r < g.R) {
        const RangeMeta m = rmeta[r];
        range_origin(g, r, rs.x0, rs.y0);
        rs.sb = m.sb;
        rs.ssb = (double)m.var / (double)g.N;
        rs.active = !m.shadow;
      }
      rs.sqrtT = rs.active ? -1e30f : 1e30f;  // inactive lanes prune everything
      rows[lane] = rs;
    }
    const bool active = rows[lane].active;
    const float sb_f = (float)rows[lane].sb;
    float sqrtT = rows[lane].sqrtT;
    double thr = rows[lane].thr;
    const uint32_t taddr = tmem_base + ((uint32_t)(quarter * 32) << 16) + (buf * 2 + sub) * kTileCols;
    int qcount = 0;  // warp-uniform

    TileMeta next_meta{{0.f, 0.f}, {0, -1}};
    if (buf < ntiles && lane < kTcTileDomains) {
      next_meta.f = meta_f[phys(t_begin + buf) * kTcTileDomains + lane];
      next_meta.i = meta_i[phys(t_begin + buf) * kTcTileDomains + lane];
    }
    // Shared pruning bar: read from L2 once per tile and applied at the next tile, so no
    // global-memory latency sits between the accumulator-full wait and the buffer release.
    unsigned long long gb_bits = ~0ull;
    for (int i = buf; i < ntiles; i += 2) {
      const uint32_t bph = (i >> 1) & 1;
      const int d0 = phys(t_begin + i) * kTcTileDomains;
      __syncwarp();
      if (lane < kTcTileDomains) {
        smeta[lane] = next_meta;
        if (i + 2 < ntiles) {  // prefetch the metadata of this group's next tile
          next_meta.f = meta_f[phys(t_begin + i + 2) * kTcTileDomains + lane];
          next_meta.i = meta_i[phys(t_begin + i + 2) * kTcTileDomains + lane];
        }
      }
      __syncwarp();
      gb_bits = (gbest && active) ? __ldcg(gbest + r) : ~0ull;
      ptx::mbar_wait(&tfull_bar[buf], bph);
      ptx::tc_fence_after();
      if ((g.flags & 32) && counters && blockIdx.x == 0 && blockIdx.y == 0 && i < 64 && lane == 0 && quarter == 0 &&
          sub == 0)
        counters[8 + 128 + i] = clock64();
      {
        const double gb = __longlong_as_double((long long)gb_bits);
        if (active && gb < thr) {
          thr = gb;
          rows[lane].thr = gb;
          sqrtT = prune_sqrtT(rows[lane].ssb, gb, NN);
          rows[lane].sqrtT = sqrtT;
        }
      }
#pragma unroll 1
      for (int h = 0; h < ((g.flags & 8) ? 0 : kTileCols / 64); ++h) {  // debug: flags&8 skips the epilogue
        __syncwarp();  // tcgen05.ld is .sync.aligned
        uint32_t v[64];
        ptx::tmem_ld_32x32b_x32(taddr + h * 64, v);
        ptx::tmem_ld_32x32b_x32(taddr + h * 64 + 32, v + 32);
        ptx::tmem_ld_wait();
        if (h == kTileCols / 64 - 1) {  // all accumulator columns are in registers: free the buffer
          ptx::tc_fence_before();
          __syncwarp();
          if (lane == 0) ptx::mbar_arrive(&tempty_bar[buf]);
          if ((g.flags & 32) && counters && blockIdx.x == 0 && blockIdx.y == 0 && i < 64 && lane == 0 &&
              quarter == 0 && sub == 0)
            counters[8 + 192 + i] = clock64();
        }
        // 8-isometry group bound for 8 domains, branch-free
        uint32_t gmask = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const float* f = reinterpret_cast<const float*>(v + 8 * j);
          // 3-input min/max chains (FMNMX3): 4 + 4 ops for the 8 isometries
          const float mx = fmaxf(fmaxf(fmaxf(fmaxf(fmaxf(fmaxf(fmaxf(f[0], f[1]), f[2]), f[3]), f[4]), f[5]), f[6]), f[7]);
          const float mn = fminf(fminf(fminf(fminf(fminf(fminf(fminf(f[0], f[1]), f[2]), f[3]), f[4]), f[5]), f[6]), f[7]);
          const DomainMetaF m = smeta[h * 8 + j].f;
          // interval [a*Sb - rad, a*Sb + rad], rad = e*sqrtT - slack, one rounding per end
          const float rad = __fmaf_rn(m.e, sqrtT, -kBoundSlack);
          const float hi = __fmaf_rn(m.a, sb_f, rad);
          const float lo = __fmaf_rn(m.a, sb_f, -rad);
          const bool keep = (mx > hi) | (mn < lo);
          gmask |= (uint32_t)keep << j;
        }
        if (g.flags & 1) gmask = active ? 0xFFu : 0u;
        if (__any_sync(0xffffffffu, gmask != 0)) {
          // push surviving groups (domain-major, lane-minor) onto the warp's queue
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            const bool mine = (gmask >> j) & 1u;
            const uint32_t bal = __ballot_sync(0xffffffffu, mine);
            if (bal == 0) continue;
            const int cnt = __popc(bal);
            if (qcount + cnt > kQCap) {
              flush_queue<NN>(queue, qcount, rows, g, meta_f, meta_i, pool, img, gbest, counters);
              qcount = 0;
              sqrtT = rows[lane].sqrtT;
              thr = rows[lane].thr;
            }
            if (mine) {
              QEntry* q = queue + qcount + __popc(bal & ((1u << lane) - 1u));
              const TileMeta& tm = smeta[h * 8 + j];
              q->d = d0 + h * 8 + j;
              q->owner = lane;
              q->a = tm.f.a;
              q->e = tm.f.e;
              q->sq = tm.i.sq;
              q->den = tm.i.den;
              *reinterpret_cast<uint4*>(q->acc) = make_uint4(v[8 * j], v[8 * j + 1], v[8 * j + 2], v[8 * j + 3]);
              *reinterpret_cast<uint4*>(q->acc + 4) = make_uint4(v[8 * j + 4], v[8 * j + 5], v[8 * j + 6], v[8 * j + 7]);
            }
            qcount += cnt;
          }
        }
      }
      if (g.flags & 8) {  // debug path skipped the loads: release here
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(&tempty_bar[buf]);
      }

      if (qcount >= 32) {
        flush_queue<NN>(queue, qcount, rows, g, meta_f, meta_i, pool, img, gbest, counters);
        qcount = 0;
        sqrtT = rows[lane].sqrtT;
        thr = rows[lane].thr;
      }
    }
    if (qcount > 0) flush_queue<NN>(queue, qcount, rows, g, meta_f, meta_i, pool, img, gbest, counters);
    __syncwarp();
    if (r < g.R) {
      const RowState& rs = rows[lane];
      partials[(long long)(blockIdx.y * 2 + buf) * g.R + r] = Partial{rs.best, rs.bd, rs.bs, rs.qs, rs.qo};
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tmem_base);
  }
}

size_t tc_smem_bytes(int K) { return tc_smem_layout(K).total; }

bool tc_supported(const Geometry& g) { return g.N == 4 || g.N == 16 || g.N == 64; }

int tc_rows_per_cta() { return kTcRows; }
int tc_tile_domains() { return kTcTileDomains; }

template <int NN>
static cudaError_t launch_tc(const unsigned char* img, const Geometry& g, const unsigned char* pool,
                             const DomainMetaF* meta_f, const DomainMetaI* meta_i, const RangeMeta* rmeta,
                             int n_chunks, int tiles_per_chunk, int tile_step, Partial* partials,
                             unsigned long long* gbest, unsigned long long* counters, cudaStream_t st) {
  const int n_tiles = (g.D_pad / kTcTileDomains + tile_step - 1) / tile_step;
  dim3 grid((g.R + kTcRows - 1) / kTcRows, n_chunks);
  const size_t smem = tc_smem_bytes(g.K);
  const cudaError_t e =
      cudaFuncSetAttribute(matcher_tc_kernel<NN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  matcher_tc_kernel<NN><<<grid, kTcThreads, smem, st>>>(img, g, pool, meta_f, meta_i, rmeta, tiles_per_chunk,
                                                        n_tiles, tile_step, partials, gbest, counters);
  return cudaGetLastError();
}

// n_chunks x tiles_per_chunk are in units of kTcTileDomains-domain tiles of the sequence
// 0, tile_step, 2*tile_step, ...
cudaError_t launch_matcher_tc(const unsigned char* img, const Geometry& g, const unsigned char* pool,
                              const DomainMetaF* meta_f, const DomainMetaI* meta_i, const RangeMeta* rmeta,
                              int n_chunks, int tiles_per_chunk, int tile_step, Partial* partials,
                              unsigned long long* gbest, unsigned long long* counters, cudaStream_t st) {
  if (g.N == 4)
    return launch_tc<4>(img, g, pool, meta_f, meta_i, rmeta, n_chunks, tiles_per_chunk, tile_step, partials, gbest,
                        counters, st);
  if (g.N == 16)
    return launch_tc<16>(img, g, pool, meta_f, meta_i, rmeta, n_chunks, tiles_per_chunk, tile_step, partials, gbest,
                         counters, st);
  return launch_tc<64>(img, g, pool, meta_f, meta_i, rmeta, n_chunks, tiles_per_chunk, tile_step, partials, gbest,
                       counters, st);
}

}  // namespace ficb
