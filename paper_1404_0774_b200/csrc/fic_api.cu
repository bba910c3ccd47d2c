// fic_api.cu — the C-ABI (include/fic_b200.h) and its host-side orchestration.
//
// Validation and error semantics follow the reference entry points they replace
// (proj/src/encoder.cpp:323-427, proj/src/decoder.cpp:39-146, proj/src/params.cpp:9-23,
// proj/src/image.cpp:138-149); all compute runs in the kernels of this directory.
// There is no CPU fallback: every failure of the CUDA runtime surfaces as FIC_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "common.cuh"

namespace ficb {
// kernels (pool.cu, matcher_*.cu, decoder.cu)
void launch_pool_build(const unsigned char*, const Geometry&, unsigned char*, DomainMetaF*, DomainMetaI*,
                       unsigned long long*, cudaStream_t);
void launch_range_pass(const unsigned char*, const Geometry&, RangeMeta*, unsigned long long*, cudaStream_t);
void launch_matcher_simt(const unsigned char*, const Geometry&, const unsigned char*, const DomainMetaF*,
                         const DomainMetaI*, const RangeMeta*, int, int, Partial*, unsigned long long*,
                         unsigned long long*, cudaStream_t);
void launch_seed(const unsigned char*, const Geometry&, const unsigned char*, const DomainMetaI*, const RangeMeta*,
                 unsigned long long*, cudaStream_t);
void launch_finalize(const unsigned char*, const Geometry&, const RangeMeta*, const Partial*, int, fic_mapping*,
                     cudaStream_t);
struct RangeXform {
  double s, o;
  int dx, dy;
  int sym;
  int pad;
};
int decode_blocks(long long);
int decode_partials(int, int, int, bool);
void launch_xform(const fic_mapping*, int, int, const Geometry&, RangeXform*, cudaStream_t);
void launch_decode_step(const double*, double*, const RangeXform*, int, int, int, int, int, double*, cudaStream_t);
void launch_rmse_finish(const double*, int, long long, double*, int, cudaStream_t);
bool decode_mean_ok(int, int, int, bool);
void launch_mean_init(double*, int, int, int, const unsigned char*, cudaStream_t);
void launch_decode_means(const double*, const double*, int, const unsigned char*, double*, const RangeXform*, int,
                         int, int, int, double*, unsigned char*, cudaStream_t);
void launch_raster_init(double*, long long, int, const unsigned char*, cudaStream_t);
void launch_quantize_raster(const double*, long long, unsigned char*, cudaStream_t);
// scan.cu (tcgen05 path, n in {2, 4, 8})
bool scan_supported(const Geometry&);
int scan_tiles(const Geometry&);
long long scan_pool_domains(const Geometry&);
void launch_pool_v3(const unsigned char*, const Geometry&, __half*, unsigned short*, DomainMetaI*,
                    unsigned long long*, RangeMeta*, unsigned long long*, void*, double*, cudaStream_t,
                    float* = nullptr, unsigned char* = nullptr, unsigned long long* = nullptr);
void launch_fill_u64(unsigned long long*, long long, unsigned long long, cudaStream_t);
void launch_seed_v3(const unsigned char*, const Geometry&, const unsigned short*, const DomainMetaI*,
                    const RangeMeta*, unsigned long long*, const double*, int, cudaStream_t);
size_t deq_table_entries(const Geometry&);
void launch_deq_tables(const Geometry&, double*, cudaStream_t);
int scan_grid(const Geometry&, int, int);
cudaError_t launch_scan(const unsigned char*, const Geometry&, int, int, const __half*, const RangeMeta*,
                        const unsigned char*, const float*, uint2*, unsigned long long*, unsigned long long, void*,
                        unsigned long long*, const unsigned short*, const DomainMetaI*, unsigned long long*, void*,
                        const double*, bool, cudaStream_t, cudaEvent_t);
bool scan_fused();
int scan_level_launches(const Geometry&, int, int, bool);
size_t scan_rec_bytes(unsigned long long, int);
int scan_trace_copy(long long*, int);
int scan_padded_ranges(const Geometry&);
void launch_threshold(const Geometry&, const RangeMeta*, const unsigned long long*, float*, cudaStream_t);
bool scan_use_f16acc(const Geometry&, int stride, int sms, bool sparse_levels);
size_t range_op_bytes(const Geometry&);
void launch_level_ops(const unsigned char*, const Geometry&, const RangeMeta*, const unsigned long long*, float*,
                      unsigned char*, unsigned long long*, bool, unsigned long long*, cudaStream_t);
void launch_eval(const unsigned char*, const Geometry&, const unsigned short*, const DomainMetaI*, const RangeMeta*,
                 const uint2*, const unsigned long long*, int, unsigned long long, double*, unsigned long long*,
                 const double*, uint2*, unsigned*, void*, bool, bool, int, cudaStream_t);
bool eval_inline();
void launch_winner(const uint2*, const unsigned long long*, int, unsigned long long, const double*,
                   const unsigned long long*, void*, int, cudaStream_t);
void launch_record(const unsigned char*, const Geometry&, const unsigned short*, const DomainMetaI*,
                   const RangeMeta*, const void*, const unsigned long long*, fic_mapping*, unsigned long long*,
                   const unsigned long long*, int, unsigned long long*, unsigned long long*, unsigned long long*,
                   unsigned long long*, int, bool, unsigned long long*, int, int, cudaStream_t);
void launch_probe_corr(const unsigned char*, const Geometry&, const unsigned short*, int, const int*, const int*,
                       const int*, long long*, cudaStream_t);
}  // namespace ficb

using namespace ficb;

namespace {

const char* const kErrcNames[] = {"MalformedHeader", "UnsupportedMaxval", "TruncatedData", "NotSquare",
                                  "NotPowerOfTwo", "IndivisibleByRange", "TooSmallForDomain", "OddSide",
                                  "SideMismatch", "OutOfBounds", "NoValidPositions", "OutOfRange",
                                  "GeometryError", "ScaleMismatch", "DimensionMismatch", "NonContractive",
                                  "BadParams", "IoError"};

thread_local std::string g_err;
std::atomic<unsigned long long> g_launches{0};
std::atomic<int> g_timing{0};
std::mutex g_timing_mu;
double g_timing_ms = 0.0;
unsigned long long g_timing_n = 0;
double g_scan_ms = 0.0;            // the full-level scan kernel alone
unsigned long long g_scan_n = 0;
double g_scan_expand_ms = 0.0;     // the full-level scan kernel + expand_kernel
double g_decode_ms = 0.0;          // decode iterations (decode_step + RMSE partials), device time
unsigned long long g_decode_n = 0;
double g_decode_bytes = 0.0;       // their algorithmic bytes
double g_pool_ms = 0.0;            // K1 pool builder, device time
unsigned long long g_pool_n = 0;
double g_pool_bytes = 0.0;         // its algorithmic bytes (image read + pool written)
std::mutex g_surv_mu;
std::vector<unsigned long long> g_last_surv;  // survivors per level of the last encode (tcgen05 path)

int32_t fail(int32_t code, const std::string& detail) {
  g_err = detail;
  return code;
}

struct CudaFail {
  cudaError_t e;
  const char* what;
};
struct InternalFail {
  const char* what;
};

#define CK(call)                                  \
  do {                                            \
    cudaError_t e_ = (call);                      \
    if (e_ != cudaSuccess) throw CudaFail{e_, #call}; \
  } while (0)

bool is_pow2(long v) { return v > 0 && (v & (v - 1)) == 0; }

// CodecParams::normalized (proj/src/params.cpp:9-23)
int32_t normalize(const fic_params* in, fic_params* out) {
  if (!in) return fail(FIC_ERR_BAD_PARAMS, "null params");
  fic_params p = *in;
  if (p.n < 2 || !is_pow2(p.n)) return fail(FIC_ERR_BAD_PARAMS, "n must be a power of two >= 2, got " + std::to_string(p.n));
  if (p.step == 0) p.step = p.n;
  if (p.step < 1) return fail(FIC_ERR_BAD_PARAMS, "step must be >= 1");
  if (p.s_bits < 1 || p.s_bits > 16) return fail(FIC_ERR_BAD_PARAMS, "s_bits must be in [1, 16]");
  if (p.o_bits < 1 || p.o_bits > 16) return fail(FIC_ERR_BAD_PARAMS, "o_bits must be in [1, 16]");
  if (!(p.s_max > 0.0)) return fail(FIC_ERR_BAD_PARAMS, "s_max must be positive");
  if (p.s_max > 65.535) return fail(FIC_ERR_BAD_PARAMS, "s_max exceeds the header's milli-precision range");
  p.s_max = (double)std::lround(p.s_max * 1000.0) / 1000.0;
  if (!(p.s_max > 0.0)) return fail(FIC_ERR_BAD_PARAMS, "s_max rounds to zero at milli precision");
  if (p.shadow_eps < 0.0) return fail(FIC_ERR_BAD_PARAMS, "shadow_eps must be non-negative");
  *out = p;
  return FIC_OK;
}

// validate_geometry (proj/src/image.cpp:138-149), params already normalised
int32_t geometry_check(int w, int h, const fic_params& p) {
  if (w != h) return fail(FIC_ERR_NOT_SQUARE, std::to_string(w) + "x" + std::to_string(h));
  if (w <= 0 || !is_pow2(w)) return fail(FIC_ERR_NOT_POWER_OF_TWO, "side " + std::to_string(w));
  if (w % p.n != 0)
    return fail(FIC_ERR_INDIVISIBLE_BY_RANGE, "side " + std::to_string(w) + ", n " + std::to_string(p.n));
  if (w < 2 * p.n)
    return fail(FIC_ERR_TOO_SMALL_FOR_DOMAIN,
                "side " + std::to_string(w) + " cannot hold a " + std::to_string(2 * p.n) + "-wide domain");
  return FIC_OK;
}

Geometry make_geometry(int w, int h, const fic_params& p) {
  Geometry g{};
  g.W = w;
  g.H = h;
  g.n = p.n;
  g.N = p.n * p.n;
  g.K = ((g.N + 15) / 16) * 16;
  g.step = p.step;
  g.PX = w >= 2 * p.n ? (w - 2 * p.n) / p.step + 1 : 0;
  g.PY = h >= 2 * p.n ? (h - 2 * p.n) / p.step + 1 : 0;
  g.D = g.PX * g.PY;
  g.D_pad = ((g.D + kDomainsPerTile - 1) / kDomainsPerTile) * kDomainsPerTile;
  g.RX = w / p.n;
  g.R = (w / p.n) * (h / p.n);
  g.row_begin = 0;
  g.single_x0 = -1;
  g.single_y0 = -1;
  const char* dbg = std::getenv("FIC_DEBUG");
  g.flags = dbg ? std::atoi(dbg) : 0;
  g.s_bits = p.s_bits;
  g.o_bits = p.o_bits;
  g.s_max = p.s_max;
  g.shadow_eps = p.shadow_eps;
  g.batch = 1;
  g.H1 = h;
  g.R1 = g.R;
  g.Dt = 0;
  return g;
}

// Growable device buffer.
struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) CK(cudaFree(p));
      p = nullptr;
      cap = 0;
      size_t want = bytes + bytes / 4 + 256;
      CK(cudaMalloc(&p, want));
      cap = want;
    }
    return p;
  }
};

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) CK(cudaFreeHost(p));
      p = nullptr;
      cap = 0;
      size_t want = bytes + bytes / 4 + 256;
      CK(cudaMallocHost(&p, want));
      cap = want;
    }
    return p;
  }
};

// One workspace per device; calls on a device serialise on its mutex.
struct Workspace {
  int device = -1;
  int sms = 148;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, ev2 = nullptr, ev3 = nullptr, ev4 = nullptr, ev5 = nullptr, ev6 = nullptr;
  bool scan_timed = false;
  double pool_bytes = 0.0;  // > 0: ev4/ev5 bracket a pool build of this many algorithmic bytes
  DevBuf img, pool, meta_f, meta_i, rmeta, partials, out, counters, xf, ra, rb, partial_sums, rmse, u8out, gbest,
      diag, scratch, mra, mrb, mrc, recs, rcounts, pendc, upool, qpool, win, list, res, scan_counts, ropnd, thr, deq, pend;
  HostBuf h_img, h_out, h_counters, h_raster, h_rmse, h_scan_counts;
  // batched host encodes: the second image / record buffers of the double-buffered pipeline and
  // the stream that uploads the next pass while the current one encodes
  DevBuf img2, out2;
  HostBuf h_img2, h_out2;
  cudaStream_t copy_stream = nullptr;
  cudaEvent_t ev_up = nullptr;
  unsigned long long list_cap = 0;        // survivor-list capacity (entries) of the current encode
  unsigned long long list_cap_grown = 0;  // capacity later encodes start from (grown on overflow)
  // CUDA graphs of the scan-path encode, keyed by everything its launches bake in
  struct Graph {
    std::vector<unsigned long long> key;
    cudaGraph_t graph = nullptr;  // kept for out_node (the records read-back, retargeted per call)
    cudaGraphNode_t out_node = nullptr;
    void* out_dst = nullptr;
    cudaGraphExec_t exec = nullptr;
    unsigned long long launches = 0;
    unsigned long long used = 0;
  };
  std::vector<Graph> graphs;
  std::vector<std::vector<unsigned long long>> seen_keys;  // fingerprints of recent eager encodes
  unsigned long long graph_clock = 0;
  void* counts_zeroed = nullptr;  // the status block whose accumulators were cleared (scan_bufs)
  // device alias of the page-locked status copy (h_scan_counts + kSelfcheckSlot): record_kernel
  // writes the status there directly (null: the status is read back by a copy)
  unsigned long long* hstat_dev = nullptr;
  std::mutex mu;
};

std::mutex g_ws_mu;
std::vector<Workspace*> g_ws;

Workspace& workspace() {
  int dev = 0;
  CK(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_ws_mu);
  if ((int)g_ws.size() <= dev) g_ws.resize(dev + 1, nullptr);
  if (!g_ws[dev]) {
    Workspace* w = new Workspace();
    w->device = dev;
    CK(cudaDeviceGetAttribute(&w->sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaStreamCreateWithFlags(&w->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&w->ev0));
    CK(cudaEventCreate(&w->ev1));
    CK(cudaEventCreate(&w->ev2));
    CK(cudaEventCreate(&w->ev3));
    CK(cudaEventCreate(&w->ev6));
    CK(cudaEventCreate(&w->ev4));
    CK(cudaEventCreate(&w->ev5));
    CK(cudaStreamCreateWithFlags(&w->copy_stream, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&w->ev_up, cudaEventDisableTiming));
    g_ws[dev] = w;
  }
  return *g_ws[dev];
}

// Split n_tiles into chunks so that m_tiles x chunks CTAs fill whole waves: minimise
// waves * (tiles per CTA + a per-CTA startup allowance).  Returns {n_chunks, tiles_per_chunk}.
std::pair<int, int> plan_chunks(int n_tiles, int m_tiles, long long wave) {
  int n_chunks = 1;
  double best_cost = 1e300;
  for (int c = 1; c <= std::min(n_tiles, 256); ++c) {
    const int tpc = (n_tiles + c - 1) / c;
    const int cc = (n_tiles + tpc - 1) / tpc;
    const long long ctas = (long long)m_tiles * cc;
    const long long waves = (ctas + wave - 1) / wave;
    const double cost = (double)waves * (tpc + 6);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      n_chunks = cc;
    }
  }
  const int tpc = (n_tiles + n_chunks - 1) / n_chunks;
  return {(n_tiles + tpc - 1) / tpc, tpc};
}

int matcher_mode(const Geometry& g) {
  const char* env = std::getenv("FIC_MATCHER");
  const bool want_simt = env && std::strcmp(env, "simt") == 0;
  return (!want_simt && scan_supported(g)) ? 1 : 0;  // 1 = tcgen05 scan (scan.cu)
}

constexpr int kMaxLevels = 6;
constexpr int kPartSlots = 512;      // per-level survivor counters, one per scan CTA (<= 2 x SMs)
// per-level survivor counters, then one status block the host reads back after every encode:
// record self-check failures, the pending count, the largest full-level partition (computed on
// the device) and the flat / shadow counters of each slice (up to 64 slices per pass)
constexpr int kSelfcheckSlot = kMaxLevels * kPartSlots;
constexpr int kPendSlot = kSelfcheckSlot + 1;
constexpr int kNeedSlot = kPendSlot + 1;
constexpr int kCounterSlot = kNeedSlot + 1;
constexpr int kAccumSlot = kCounterSlot + 2 * 64;  // flat / shadow accumulators (pool launch atomics)
constexpr int kTicketSlot = kAccumSlot + 2 * 64;   // record_kernel's last-block ticket
constexpr int kScanCountSlots = kTicketSlot + 2;

// Scan levels: sparse passes over every 8^k-th (or 4 * 8^k-th) 128-domain tile seed the
// pruning bar, then the full scan.  Each level prunes with the bar the previous
// ones achieved, so survivors per level stay near (level size / previous level size) x the
// handful of candidates whose bound is within the quantisation slack of the optimum.
std::vector<int> scan_levels(const Geometry& g) {
  std::vector<int> lv;
  const int tiles = scan_tiles(g);
  const char* pp = std::getenv("FIC_PREPASS");
  const bool prepass = !(pp && std::strcmp(pp, "0") == 0);
  // large pools: ratio 8 between levels, the last sparse level at stride 16 (cfg4 with the fp16
  // full level: {4096, 512, 64, 16} 65.1-65.4 ms vs {..., 8} 67.5-68.0, alternated on one box:
  // the stride-8 level's 10.8 ms of hit-heavy selection cost more than its bar saves at the
  // full level; 3 or 5 levels are no better: 68.3 / 64.3 ms)
  const char* sched = std::getenv("FIC_LEVELS");  // optional override, e.g. "64,8"
  if (sched) {
    for (const char* p = sched; *p;) {
      const int v = std::atoi(p);
      if (v > 1 && tiles > v) lv.push_back(v);
      while (*p && *p != ',') ++p;
      if (*p == ',') ++p;
    }
  } else if (prepass && tiles > 1024) {
    for (int s : {4096, 512, 64, 16})
      if (tiles > s) lv.push_back(s);
  } else if (prepass) {
    // small pools (cfg2: 123 tiles, cfg3: 501): last sparse level at stride 4, earlier ones x8
    // while they keep >= 8 tiles.  The sparse levels evaluate only each warp's best column per
    // range (scan_kernel, lv.select), so they are cheap and a denser last level pays off
    // (measured: cfg2 {4} 0.56 ms vs {64, 8} 0.61; cfg3 {32, 4} 3.09 vs {64, 8} 3.65).
    std::vector<int> rev;
    for (int s = 4; tiles >= 8 * s; s *= 8) rev.push_back(s);
    // a last level short enough for per-lane bests at stride 3 (<= 48 level tiles) gives a
    // better bar for a few more tiles: cfg2 {3} 0.271 vs {4} 0.278 ms (cfg3's stride-4 level
    // is hit-first; {32, 3} there measured slower)
    if (!rev.empty() && (tiles + 2) / 3 <= 48) rev[0] = 3;
    // pools too small for a stride-4 level with 8 tiles still get one at stride 3 (from 6
    // tiles): its per-lane bests give the full level a bar the local seed cannot (cfg1, 30
    // tiles: 0.233 -> 0.101 ms)
    if (rev.empty() && tiles >= 6) rev.push_back(3);
    lv.assign(rev.rbegin(), rev.rend());
  }
  // the host keeps kMaxLevels counter partitions (sparse levels + the full one): an override
  // with more levels keeps its last (densest) kMaxLevels - 1 sparse levels
  if (lv.size() > (size_t)kMaxLevels - 1) lv.erase(lv.begin(), lv.end() - (kMaxLevels - 1));
  lv.push_back(1);
  return lv;
}

struct ScanBufs {
  __half* upool;
  unsigned short* qpool;
  DomainMetaI* mi;
  RangeMeta* rm;
  unsigned long long* gbest;
  void* win;  // per range: 128-bit (residual bits, domain * 8 + isometry) minimum
  unsigned long long* cnt;
  unsigned char* ropnd;
  float* thr;
  double* deq;
};

ScanBufs scan_bufs(Workspace& ws, const Geometry& g) {
  const long long Dt = (long long)g.Dt * g.batch;  // every slice's pool
  ScanBufs b;
  b.upool = static_cast<__half*>(ws.upool.get((size_t)Dt * g.K * 2));
  b.qpool = static_cast<unsigned short*>(ws.qpool.get((size_t)Dt * 8 * g.N * 2));  // q8: [domain][isometry][N]
  b.mi = static_cast<DomainMetaI*>(ws.meta_i.get((size_t)Dt * sizeof(DomainMetaI)));
  b.rm = static_cast<RangeMeta*>(ws.rmeta.get((size_t)g.R * sizeof(RangeMeta)));
  b.gbest = static_cast<unsigned long long*>(ws.gbest.get((size_t)g.R * sizeof(unsigned long long)));
  b.win = ws.win.get((size_t)g.R * 16);
  b.ropnd = static_cast<unsigned char*>(ws.ropnd.get(range_op_bytes(g)));
  // thresholds, then one allpass bit mask per 32-range m-tile
  b.thr = static_cast<float*>(ws.thr.get((size_t)scan_padded_ranges(g) * sizeof(float) * 33 / 32));
  b.deq = static_cast<double*>(ws.deq.get(deq_table_entries(g) * sizeof(double)));
  b.cnt = static_cast<unsigned long long*>(ws.scan_counts.get(kScanCountSlots * sizeof(unsigned long long)));
  if (ws.scan_counts.p != ws.counts_zeroed) {  // new status block: clear the accumulators and the ticket once
    CK(cudaMemsetAsync(b.cnt + kAccumSlot, 0, (kScanCountSlots - kAccumSlot) * sizeof(unsigned long long), ws.stream));
    CK(cudaStreamSynchronize(ws.stream));
    ws.counts_zeroed = ws.scan_counts.p;
  }
  return b;
}

// One scan level: tensor-core scan appending survivors to per-CTA list partitions, then
// their exact evaluation.  cnt: the level's kPartSlots counters.
void enqueue_level(Workspace& ws, const unsigned char* d_img, const Geometry& g, const ScanBufs& b, int stride,
                   unsigned long long* cnt, cudaStream_t st, bool ops_prebuilt = false) {
  auto* list = static_cast<uint2*>(ws.list.get((size_t)ws.list_cap * sizeof(uint2)));
  auto* res = static_cast<double*>(ws.res.get((size_t)ws.list_cap * sizeof(double)));
  const int parts = scan_grid(g, stride, ws.sms);
  // pending list: one segment per eval block (sized for the largest level grid, so the buffer
  // does not move between levels)
  // (blocks x segment <= list_cap + parts x 2048 for any parts <= kPartSlots)
  auto* pend = static_cast<uint2*>(ws.pend.get((ws.list_cap + (size_t)kPartSlots * 2048) * sizeof(uint2)));
  auto* pendc = static_cast<unsigned*>(ws.pendc.get((size_t)kPartSlots * 8 * sizeof(unsigned)));
  const unsigned long long part = ws.list_cap / (unsigned long long)parts;
  const bool final_level = stride == 1;  // resets the winner slots and the self-check counter too
  // the full level accumulates in fp16 after sparse levels or for large pools (flags & 256: its
  // thresholds and its scan)
  Geometry gl = g;
  gl.flags = scan_use_f16acc(g, stride, ws.sms, scan_levels(g).size() > 1) ? (g.flags | 256) : (g.flags & ~256);
  // (the first level of an encode without a seed: built by the pool launch, no bar yet)
  if (!ops_prebuilt)
    launch_level_ops(d_img, gl, b.rm, b.gbest, b.thr, b.ropnd, b.cnt + kPendSlot, final_level,
                     final_level ? b.cnt + kSelfcheckSlot : nullptr, st);
  const bool time_scan = stride == 1 && g_timing.load() != 0;
  if (time_scan) CK(cudaEventRecord(ws.ev2, st));
  void* recs = ws.recs.get(scan_rec_bytes(ws.list_cap, parts));
  auto* rcnt = static_cast<unsigned long long*>(ws.rcounts.get(kPartSlots * sizeof(unsigned long long)));
  const bool fused = scan_fused();
  CK(launch_scan(d_img, gl, stride, ws.sms, b.upool, b.rm, b.ropnd, b.thr, list, cnt, part, recs, rcnt, b.qpool,
                 b.mi, b.gbest, b.win, b.deq, fused, st, time_scan ? ws.ev6 : nullptr));
  if (time_scan) {
    CK(cudaEventRecord(ws.ev3, st));
    ws.scan_timed = true;
  }
  g_launches += (ops_prebuilt ? 0 : 1) + scan_level_launches(g, stride, ws.sms, fused);  // level ops, scan (+ expand)
  if (fused) return;  // the scan evaluated its survivors itself
  const bool inl = eval_inline();
  // sparse levels only lower the bar: closed-form upper bounds (FIC_SPARSE_EXACT=1: exact residuals)
  const char* se = std::getenv("FIC_SPARSE_EXACT");
  const bool bar_only = !final_level && !(se && se[0] == '1');
  launch_eval(d_img, g, b.qpool, b.mi, b.rm, list, cnt, parts, part, res, b.gbest, b.deq, pend,
              pendc, b.win, inl, bar_only, ws.sms, st);
  g_launches += inl || bar_only ? 1 : 2;  // evaluation (+ residuals)
}

// The full level plus winner selection and records.  Its list must be complete; a
// truncated one (count > cap) is detected by the caller, which re-runs this part only.
// snapshot: the record kernel moves the flat / shadow accumulators to the status slots (false
// on a re-run of the full level after an overflow: the first run's snapshot stands).
void enqueue_final(Workspace& ws, const unsigned char* d_img, const Geometry& g, const ScanBufs& b, size_t level,
                   fic_mapping* d_out, cudaStream_t st, bool snapshot = true) {
  unsigned long long* cnt = b.cnt + level * kPartSlots;
  enqueue_level(ws, d_img, g, b, 1, cnt, st);
  const bool timed = g_timing.load() != 0;
  if (timed) CK(cudaEventRecord(ws.ev1, st));
  const int parts = scan_grid(g, 1, ws.sms);
  if (!scan_fused() && !eval_inline()) {
    launch_winner(static_cast<uint2*>(ws.list.p), cnt, parts, ws.list_cap / (unsigned long long)parts,
                  static_cast<double*>(ws.res.p), b.gbest, b.win, ws.sms, st);
    g_launches += 1;
  }
  launch_record(d_img, g, b.qpool, b.mi, b.rm, b.win, b.gbest, d_out, b.cnt + kSelfcheckSlot, cnt, parts,
                b.cnt + kNeedSlot, b.cnt + kAccumSlot, b.cnt + kCounterSlot, b.cnt + kTicketSlot, 2 * g.batch, snapshot,
                ws.hstat_dev, kNeedSlot - kSelfcheckSlot, kCounterSlot - kSelfcheckSlot, st);
  g_launches += 1;
  CK(cudaGetLastError());
}

// tcgen05 path: K1 normalised pool, range pass, seed, sparse levels, final level.
void enqueue_encode_scan(Workspace& ws, const unsigned char* d_img, const Geometry& g, const ScanBufs& b,
                         fic_mapping* d_out, unsigned long long* d_counters, cudaStream_t st) {
  // list capacity: the geometry's default, or what an earlier overflow grew it to
  ws.list_cap_grown = std::max(ws.list_cap_grown, std::max<unsigned long long>(1ull << 22, (unsigned long long)g.R * 8 * 128));
  ws.list_cap = ws.list_cap_grown;
  if (const char* lc = std::getenv("FIC_LIST_CAP")) ws.list_cap = std::strtoull(lc, nullptr, 10);  // tests: force overflow
  // b.cnt: the scan kernels write their partitions' counters, range_op resets the pending and
  // self-check slots, the host reads only the partitions a level used; the flat / shadow counts
  // accumulate in the kAccumSlot slots, which record_kernel moves to d_counters (the kCounterSlot
  // slots) and clears for the next encode (zeroed once when the block is allocated, scan_bufs)
  (void)d_counters;
  const bool time_pool = g_timing.load() != 0;
  // The local seed gives the first scan level a bar (upper bounds of the range's 3 x 3 local
  // self-similar candidates) for large pools.  Small pools (<= 1024 tiles) start with a
  // per-lane-best selection level that keeps nearly every lane's best column whatever the bar,
  // so they skip it: cfg2 0.335 / 0.337 / 0.344 ms without / with a 1 x 1 / 3 x 3 seed, cfg3
  // 2.456 / 2.447 / 2.462 ms (within noise), one launch fewer.  FIC_SEED=0 / 1 / 3 forces none /
  // 1 x 1 / 3 x 3.
  // Without any sparse level (pools under 6 tiles) the seed is the full level's only bar.
  const char* seed_env = std::getenv("FIC_SEED");
  const int seed_side =
      seed_env ? std::atoi(seed_env) : (scan_tiles(g) > 1024 || scan_levels(g).size() == 1 ? 3 : 0);
  const bool seed = seed_side > 0;
  const std::vector<int> lv = scan_levels(g);
  // without a seed the first (sparse) level scans with no bar: its range operands do not depend
  // on any evaluation and are built by the pool launch (one launch fewer; FIC_PREOPS=0: off)
  const char* pre_env = std::getenv("FIC_PREOPS");
  const bool pre_ops = !seed && lv.size() > 1 && lv[0] != 1 && !(pre_env && pre_env[0] == '0');
  if (time_pool) CK(cudaEventRecord(ws.ev4, st));
  // K1 pool + range pass + bar / winner init + dequantised tables (+ the first level's range
  // operands) in one launch
  launch_pool_v3(d_img, g, b.upool, b.qpool, b.mi, b.cnt + kAccumSlot, b.rm, b.gbest, b.win, b.deq, st,
                 pre_ops ? b.thr : nullptr, pre_ops ? b.ropnd : nullptr, pre_ops ? b.cnt + kPendSlot : nullptr);
  if (time_pool) {
    CK(cudaEventRecord(ws.ev5, st));
    // algorithmic bytes: the image read once, the pool written once (fp16 operand 2K, exact
    // cells 8 x N u16, meta 16 B per padded domain), and the preparations riding in the same
    // launch: per range its N pixels read, RangeMeta (16 B), bar (8 B) and winner key (16 B)
    const double Dt = (double)g.Dt * g.batch;
    ws.pool_bytes = (double)g.W * g.H + Dt * (2.0 * g.K + 16.0 * g.N + 16.0) + (double)g.R * (g.N + 40.0);
    // the first level's range operands (8 rows of K fp16 per range) and thresholds
    if (pre_ops) ws.pool_bytes += (double)g.R * (16.0 * g.K + 4.0);
  }
  if (seed) launch_seed_v3(d_img, g, b.qpool, b.mi, b.rm, b.gbest, b.deq, seed_side >= 3 ? 1 : 0, st);
  g_launches += seed ? 2 : 1;
  if (g_timing.load()) CK(cudaEventRecord(ws.ev0, st));
  for (size_t l = 0; l + 1 < lv.size(); ++l)
    enqueue_level(ws, d_img, g, b, lv[l], b.cnt + l * kPartSlots, st, l == 0 && pre_ops);
  enqueue_final(ws, d_img, g, b, lv.size() - 1, d_out, st);
}

// n >= 16 path (and FIC_MATCHER=simt): 8-isometry fp16 pool + CUDA-core matcher
// (matcher_simt.cu), exact integer correlations.
void enqueue_encode_simt(Workspace& ws, const unsigned char* d_img, const Geometry& g, fic_mapping* d_out,
                         unsigned long long* d_counters, cudaStream_t st) {
  auto* pool = static_cast<unsigned char*>(ws.pool.get((size_t)g.D_pad * g.K * 16));
  auto* mf = static_cast<DomainMetaF*>(ws.meta_f.get((size_t)g.D_pad * sizeof(DomainMetaF)));
  auto* mi = static_cast<DomainMetaI*>(ws.meta_i.get((size_t)g.D_pad * sizeof(DomainMetaI)));
  auto* rm = static_cast<RangeMeta*>(ws.rmeta.get((size_t)g.R * sizeof(RangeMeta)));
  const int rows_per_cta = 128;
  const int n_tiles = g.D_pad / kDomainsPerTile;
  const int m_tiles = (g.R + rows_per_cta - 1) / rows_per_cta;
  const std::pair<int, int> plan = plan_chunks(n_tiles, m_tiles, (long long)ws.sms * 8);
  const int n_chunks = plan.first, tiles_per_chunk = plan.second;
  auto* parts = static_cast<Partial*>(ws.partials.get((size_t)n_chunks * g.R * sizeof(Partial)));
  auto* gbest = static_cast<unsigned long long*>(ws.gbest.get((size_t)g.R * sizeof(unsigned long long)));
  unsigned long long* diag = nullptr;
  if (g.flags & 4) {
    diag = static_cast<unsigned long long*>(ws.diag.get((8 + 256) * sizeof(unsigned long long)));
    CK(cudaMemsetAsync(diag, 0, (8 + 256) * sizeof(unsigned long long), st));
  }
  CK(cudaMemsetAsync(d_counters, 0, 2 * sizeof(unsigned long long), st));
  launch_pool_build(d_img, g, pool, mf, mi, d_counters, st);
  launch_range_pass(d_img, g, rm, d_counters + 1, st);
  launch_seed(d_img, g, pool, mi, rm, gbest, st);
  const bool timed = g_timing.load() != 0;
  if (timed) CK(cudaEventRecord(ws.ev0, st));
  launch_matcher_simt(d_img, g, pool, mf, mi, rm, n_chunks, tiles_per_chunk, parts, gbest, diag, st);
  if (timed) CK(cudaEventRecord(ws.ev1, st));
  launch_finalize(d_img, g, rm, parts, n_chunks, d_out, st);
  CK(cudaGetLastError());
  g_launches += 5;
  if (diag) {
    unsigned long long h[8 + 256];
    CK(cudaMemcpyAsync(h, diag, sizeof h, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    std::fprintf(stderr, "[fic diag] simt R=%d D=%d chunks=%d groups=%llu survive=%llu tight=%llu exact=%llu\n", g.R,
                 g.D, n_chunks, h[0], h[1], h[2], h[3]);
  }
}

// The scan-path encode as a CUDA graph: ~30 dependent launches, memsets and event records
// per encode cost ~2 us of launch gap each when enqueued one by one.  The graph bakes in
// the geometry, every buffer pointer, the list capacity, the stream and the switches read
// from the environment, so those form its key; a key seen on two consecutive encodes is
// captured (the first run allocated every buffer, so capture performs no allocation) and
// replayed from then on.  FIC_NO_GRAPH=1, and encodes timed with fic_set_matcher_timing,
// enqueue eagerly.
std::vector<unsigned long long> encode_key(Workspace& ws, const unsigned char* d_img, const Geometry& g,
                                           const fic_mapping* d_out, const unsigned long long* d_counters,
                                           cudaStream_t st) {
  std::vector<unsigned long long> k;
  const int gi[] = {g.W, g.H, g.n, g.N, g.K, g.step, g.PX, g.PY, g.D, g.D_pad, g.RX, g.R, g.row_begin,
                    g.single_x0, g.single_y0, g.flags, g.s_bits, g.o_bits, g.batch, g.H1, g.R1, g.Dt};
  for (int v : gi) k.push_back((unsigned long long)(unsigned)v);
  unsigned long long bits;
  std::memcpy(&bits, &g.s_max, 8);
  k.push_back(bits);
  std::memcpy(&bits, &g.shadow_eps, 8);
  k.push_back(bits);
  (void)st;  // graphs are stream-independent (captured on the workspace stream, launched on any)
  const void* ptrs[] = {d_img, d_out, d_counters, ws.upool.p, ws.qpool.p, ws.meta_i.p, ws.rmeta.p, ws.gbest.p,
                        ws.win.p, ws.ropnd.p, ws.thr.p, ws.deq.p, ws.scan_counts.p, ws.list.p, ws.res.p, ws.pend.p,
                        ws.recs.p, ws.rcounts.p, ws.pendc.p};
  for (const void* q : ptrs) k.push_back((unsigned long long)(uintptr_t)q);
  k.push_back(ws.list_cap);
  for (const char* name : {"FIC_LEVELS", "FIC_PREPASS", "FIC_SELECT", "FIC_MATCHER", "FIC_COARSE", "FIC_SEED",
                           "FIC_LANEBEST_MAX", "FIC_F16ACC", "FIC_F16SEL", "FIC_FUSED", "FIC_EVAL_SPLIT",
                           "FIC_SPARSE_EXACT", "FIC_LANE_GROUP", "FIC_EVAL_PER", "FIC_ROTATE", "FIC_PREOPS"}) {
    const char* e = std::getenv(name);
    unsigned long long h = 1469598103934665603ull;
    for (const char* c = e ? e : "\x01"; *c; ++c) h = (h ^ (unsigned char)*c) * 1099511628211ull;
    k.push_back(h);
  }
  return k;
}

// The read-back of an encode: the status block from the self-check slot on (self-check,
// largest partition, flat / shadow counters) into the pinned `hc`, and for a host-API encode the
// records into the pinned `h_out`.
struct Readback {
  unsigned long long* hc;
  size_t status_bytes;
  fic_mapping* h_out;  // null: records stay on the device
  size_t out_bytes;
};

void enqueue_readback(const Readback& rb, const ScanBufs& b, const fic_mapping* d_out, cudaStream_t st) {
  if (rb.status_bytes)  // (0: record_kernel wrote the status into the page-locked copy itself)
    CK(cudaMemcpyAsync(rb.hc + kSelfcheckSlot, b.cnt + kSelfcheckSlot, rb.status_bytes, cudaMemcpyDeviceToHost, st));
  if (rb.h_out) CK(cudaMemcpyAsync(rb.h_out, d_out, rb.out_bytes, cudaMemcpyDeviceToHost, st));
}

// Returns true when the read-back rode in the replayed graph (its last nodes: no gap between
// the last kernel and the copies, 2 fewer host calls); false when the caller must enqueue it.
bool enqueue_encode_graph(Workspace& ws, const unsigned char* d_img, const Geometry& g, const ScanBufs& b,
                          fic_mapping* d_out, unsigned long long* d_counters, cudaStream_t st,
                          const Readback* rb) {
  if (std::getenv("FIC_NO_GRAPH") || g_timing.load()) {  // timed encodes (event records) run eagerly
    enqueue_encode_scan(ws, d_img, g, b, d_out, d_counters, st);
    return false;
  }
  // the list capacity this encode will use (as enqueue_encode_scan sets it)
  ws.list_cap_grown = std::max(ws.list_cap_grown, std::max<unsigned long long>(1ull << 22, (unsigned long long)g.R * 8 * 128));
  ws.list_cap = ws.list_cap_grown;
  if (const char* lc = std::getenv("FIC_LIST_CAP")) ws.list_cap = std::strtoull(lc, nullptr, 10);
  std::vector<unsigned long long> key = encode_key(ws, d_img, g, d_out, d_counters, st);
  key.push_back(rb ? (unsigned long long)(uintptr_t)rb->hc : 0ull);
  key.push_back(rb ? rb->status_bytes : 0ull);
  key.push_back(rb && rb->h_out ? rb->out_bytes : 0ull);
  ++ws.graph_clock;
  for (auto& gr : ws.graphs) {
    if (gr.key == key) {
      if (gr.out_node && rb->h_out != gr.out_dst) {  // retarget the records copy to this call's buffer
        CK(cudaGraphExecMemcpyNodeSetParams1D(gr.exec, gr.out_node, rb->h_out, d_out, rb->out_bytes,
                                              cudaMemcpyDeviceToHost));
        gr.out_dst = rb->h_out;
      }
      CK(cudaGraphLaunch(gr.exec, st));
      g_launches += gr.launches;
      gr.used = ws.graph_clock;
      return rb != nullptr;
    }
  }
  // first sighting: eager (allocates); capture on the next one.  A few recent keys are kept, so
  // encodes alternating between buffers (the batched pipeline) are captured too.
  if (std::find(ws.seen_keys.begin(), ws.seen_keys.end(), key) == ws.seen_keys.end()) {
    enqueue_encode_scan(ws, d_img, g, b, d_out, d_counters, st);
    std::vector<unsigned long long> k2 = encode_key(ws, d_img, g, d_out, d_counters, st);  // (buffers may have grown)
    k2.push_back(rb ? (unsigned long long)(uintptr_t)rb->hc : 0ull);
    k2.push_back(rb ? rb->status_bytes : 0ull);
    k2.push_back(rb && rb->h_out ? rb->out_bytes : 0ull);
    ws.seen_keys.push_back(std::move(k2));
    if (ws.seen_keys.size() > 4) ws.seen_keys.erase(ws.seen_keys.begin());
    return false;
  }
  const unsigned long long l0 = g_launches.load();
  cudaGraph_t graph = nullptr;
  // captured on the workspace's own stream (the caller's may be the legacy default stream,
  // which cannot be captured); nothing executes during capture
  CK(cudaStreamBeginCapture(ws.stream, cudaStreamCaptureModeRelaxed));
  try {
    enqueue_encode_scan(ws, d_img, g, b, d_out, d_counters, ws.stream);
    if (rb) enqueue_readback(*rb, b, d_out, ws.stream);
  } catch (...) {
    cudaStreamEndCapture(ws.stream, &graph);
    if (graph) cudaGraphDestroy(graph);
    throw;
  }
  CK(cudaStreamEndCapture(ws.stream, &graph));
  Workspace::Graph gr;
  gr.key = key;
  gr.launches = g_launches.load() - l0;
  gr.used = ws.graph_clock;
  gr.graph = graph;
  if (rb && rb->h_out) {  // the records copy: the memcpy node writing h_out
    size_t nn = 0;
    CK(cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    CK(cudaGraphGetNodes(graph, nodes.data(), &nn));
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType t;
      CK(cudaGraphNodeGetType(nd, &t));
      if (t != cudaGraphNodeTypeMemcpy) continue;
      cudaMemcpy3DParms mp{};
      CK(cudaGraphMemcpyNodeGetParams(nd, &mp));
      if (mp.dstPtr.ptr == rb->h_out) gr.out_node = nd;
    }
    if (!gr.out_node) throw InternalFail{"graph capture: records read-back node not found"};
    gr.out_dst = rb->h_out;
  }
  CK(cudaGraphInstantiate(&gr.exec, graph, 0));
  CK(cudaGraphLaunch(gr.exec, st));
  if (ws.graphs.size() >= 16) {  // evict the least recently used
    auto it = std::min_element(ws.graphs.begin(), ws.graphs.end(),
                               [](const Workspace::Graph& a, const Workspace::Graph& c) { return a.used < c.used; });
    CK(cudaGraphExecDestroy(it->exec));
    CK(cudaGraphDestroy(it->graph));
    ws.graphs.erase(it);
  }
  ws.graphs.push_back(std::move(gr));
  return rb != nullptr;
}

// Enqueue the whole encode of the region described by g and wait for it; a survivor list
// that overflowed is grown to the count the scan reported and the encode is re-run.
// counters[b] = flat domains and counters[batch + b] = shadow ranges of slice b (copied to
// h_counters; batch == 1 for a single image).
void run_encode(Workspace& ws, const unsigned char* d_img, const Geometry& g_in, fic_mapping* d_out,
                unsigned long long* d_counters, unsigned long long* h_counters, cudaStream_t st,
                fic_mapping* h_out = nullptr, const std::function<void()>& overlap = {}) {
  // overlap: host work run once while this encode executes (before its synchronisation)
  // h_out: the records are also copied to this (pinned) host buffer before the one synchronisation
  // (again after an overflow re-run), so a host-API encode waits for the device once
  Geometry g = g_in;
  if (g.Dt == 0) g.Dt = (int)scan_pool_domains(g);  // per-slice pool stride (a multiple of the pool block)
  if (matcher_mode(g) == 0) {
    if (g.batch != 1) throw InternalFail{"batched encode needs the tcgen05 scan path"};
    enqueue_encode_simt(ws, d_img, g, d_out, d_counters, st);
    if (h_counters)
      CK(cudaMemcpyAsync(h_counters, d_counters, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    if (h_out) CK(cudaMemcpyAsync(h_out, d_out, (size_t)g.R * sizeof(fic_mapping), cudaMemcpyDeviceToHost, st));
    if (overlap) overlap();
    CK(cudaStreamSynchronize(st));
    return;
  }
  const ScanBufs b = scan_bufs(ws, g);
  const size_t nl = scan_levels(g).size();
  auto* hc = static_cast<unsigned long long*>(ws.h_scan_counts.get(kScanCountSlots * sizeof(unsigned long long)));
  if (g.batch > 64) throw InternalFail{"more than 64 slices in one encode pass"};
  d_counters = b.cnt + kCounterSlot;  // flat / shadow counters live in the status block
  // every level's partition counters only for the survivor statistics (timed / diagnostic encodes)
  const bool all_counts = g_timing.load() != 0 || (g.flags & 4);
  // the status tail straight from record_kernel into hc (mapped page-locked memory) unless this
  // encode reads the whole block back anyway
  {
    unsigned long long* dev = nullptr;
    if (!all_counts && !std::getenv("FIC_STATUS_COPY") &&
        cudaHostGetDevicePointer(reinterpret_cast<void**>(&dev), hc + kSelfcheckSlot, 0) != cudaSuccess) {
      (void)cudaGetLastError();
      dev = nullptr;
    }
    ws.hstat_dev = all_counts ? nullptr : dev;
  }
  const Readback rb{hc, ws.hstat_dev ? 0 : (kCounterSlot - kSelfcheckSlot + 2 * g.batch) * sizeof(unsigned long long),
                    h_out, (size_t)g.R * sizeof(fic_mapping)};
  const bool in_graph = enqueue_encode_graph(ws, d_img, g, b, d_out, d_counters, st, all_counts ? nullptr : &rb);
  for (int attempt = 0;; ++attempt) {
    // one read-back of the status block (and the records of a host-API encode), one synchronisation
    if (all_counts)
      CK(cudaMemcpyAsync(hc, b.cnt, kScanCountSlots * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
    if (all_counts ? h_out != nullptr : !(attempt == 0 && in_graph)) {
      if (all_counts)
        CK(cudaMemcpyAsync(h_out, d_out, rb.out_bytes, cudaMemcpyDeviceToHost, st));
      else
        enqueue_readback(rb, b, d_out, st);
    }
    if (attempt == 0 && overlap) overlap();
    CK(cudaStreamSynchronize(st));
    if (h_counters) std::memcpy(h_counters, hc + kCounterSlot, 2 * g.batch * sizeof(unsigned long long));
    const std::vector<int> lv = scan_levels(g);
    const int fparts = scan_grid(g, 1, ws.sms);
    const unsigned long long need = hc[kNeedSlot];  // largest partition of the full level (record_kernel)
    if (g.flags & 4) {
      std::fprintf(stderr, "[fic diag] scan R=%d D=%d tiles=%d levels", g.R, g.D, scan_tiles(g));
      for (size_t l = 0; l < nl; ++l) {
        unsigned long long tot = 0, mx = 0;
        const int parts = scan_grid(g, lv[l], ws.sms);
        for (int c = 0; c < parts; ++c) {
          tot += hc[l * kPartSlots + c];
          mx = std::max(mx, hc[l * kPartSlots + c]);
        }
        std::fprintf(stderr, " %d:%llu(max part %llu)", lv[l], tot, mx);
      }
      std::fprintf(stderr, " part %llu selfcheck %llu\n", ws.list_cap / fparts, hc[kSelfcheckSlot]);
    }
    if (all_counts) {
      std::vector<unsigned long long> surv(nl, 0);
      for (size_t l = 0; l < nl; ++l) {
        const int parts = scan_grid(g, lv[l], ws.sms);
        for (int c = 0; c < parts; ++c) surv[l] += hc[l * kPartSlots + c];
      }
      std::lock_guard<std::mutex> lock(g_surv_mu);
      g_last_surv = surv;
    }
    if (need <= ws.list_cap / (unsigned long long)fparts) {
      // (debug flags 8/16/128 skip the test, the MMAs or the TMEM reads: meaningless codes)
      if (hc[kSelfcheckSlot] != 0 && !(g.flags & (8 | 16 | 128)))
        throw InternalFail{"scan self-check: a winner's residual differs from its bar"};
      return;
    }
    // a partition of the full level's list was truncated: re-run that level with a larger
    // list.  The entries evaluated so far already lowered the bar, so every attempt has
    // fewer survivors; the list grows toward the need within a quarter of free device memory.
    if (attempt >= 12) throw InternalFail{"survivor list keeps overflowing"};
    {
      const unsigned long long want = (need + need / 4 + 1024) * (unsigned long long)fparts;
      size_t free_b = 0, total_b = 0;
      CK(cudaMemGetInfo(&free_b, &total_b));
      // list + pending + residual, + the scan's mask records (40 B per two entry slots)
      // (the pending list also carries kPartSlots x 2048 slack entries, allocated on top)
      const unsigned long long per_entry = sizeof(uint2) * 2 + sizeof(double) + 20;
      const unsigned long long limit = (ws.list.cap + ws.res.cap + ws.pend.cap + ws.recs.cap + free_b / 4) / per_entry;
      ws.list_cap = std::max(ws.list_cap, std::min(want, limit));
      if (!std::getenv("FIC_LIST_CAP")) ws.list_cap_grown = ws.list_cap;
    }
    enqueue_final(ws, d_img, g, b, nl - 1, d_out, st, false);
  }
}

void collect_timing(Workspace& ws) {
  if (!g_timing.load()) return;
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, ws.ev0, ws.ev1) == cudaSuccess) {
    std::lock_guard<std::mutex> lock(g_timing_mu);
    g_timing_ms += ms;
    g_timing_n += 1;
  }
  float ms2 = 0.f;
  if (ws.scan_timed && cudaEventElapsedTime(&ms, ws.ev2, ws.ev6) == cudaSuccess &&
      cudaEventElapsedTime(&ms2, ws.ev2, ws.ev3) == cudaSuccess) {
    std::lock_guard<std::mutex> lock(g_timing_mu);
    g_scan_ms += ms;
    g_scan_expand_ms += ms2;
    g_scan_n += 1;
  }
  ws.scan_timed = false;
  if (ws.pool_bytes > 0 && cudaEventElapsedTime(&ms, ws.ev4, ws.ev5) == cudaSuccess) {
    std::lock_guard<std::mutex> lock(g_timing_mu);
    g_pool_ms += ms;
    g_pool_n += 1;
    g_pool_bytes += ws.pool_bytes;
  }
  ws.pool_bytes = 0.0;
}

// EncodeStats summed over the slices of a batch (flat[b] = h[b], shadow[b] = h[batch + b]).
void fill_stats_batch(fic_stats* stats, const Geometry& g, const unsigned long long* h) {
  if (!stats) return;
  fic_stats t{0, 0, 0};
  for (int b = 0; b < g.batch; ++b) {
    const unsigned long long flat = h[b], shadow = h[g.batch + b];
    const unsigned long long active = (unsigned long long)g.R1 - shadow;
    t.candidates_tested += 8ull * active * ((unsigned long long)g.D - flat);
    t.shadow_ranges += shadow;
    t.shadow_codeblocks += 8ull * active * flat;
  }
  *stats = t;
}

// Slices stacked into one encode pass: up to 64 when the tcgen05 scan applies and a slice
// holds whole 32-range scan tiles (so no tile straddles two slices' domain pools), else 1.
int batch_chunk(const Geometry& g) {
  if (matcher_mode(g) != 1 || g.R % 32 != 0) return 1;
  if (const char* e = std::getenv("FIC_BATCH_CHUNK")) return std::min(64, std::max(1, std::atoi(e)));
  return 64;
}

Geometry batch_geometry(const Geometry& g1, int slices) {
  Geometry g = g1;
  if (slices <= 1) return g;
  g.batch = slices;
  g.H1 = g1.H;
  g.R1 = g1.R;
  g.H = g1.H * slices;
  g.R = g1.R * slices;
  g.Dt = (int)scan_pool_domains(g1);
  return g;
}

void fill_stats(fic_stats* stats, const Geometry& g, unsigned long long flat, unsigned long long shadow) {
  if (!stats) return;
  const unsigned long long active = (unsigned long long)g.R - shadow;
  stats->candidates_tested = 8ull * active * ((unsigned long long)g.D - flat);
  stats->shadow_ranges = shadow;
  stats->shadow_codeblocks = 8ull * active * flat;
}

template <class F>
int32_t guarded(F&& f) {
  try {
    return f();
  } catch (const CudaFail& c) {
    return fail(FIC_ERR_CUDA, std::string(cudaGetErrorName(c.e)) + " (" + cudaGetErrorString(c.e) + ") at " + c.what);
  } catch (const InternalFail& f) {
    return fail(FIC_ERR_INTERNAL, f.what);
  } catch (const std::bad_alloc&) {
    return fail(FIC_ERR_INTERNAL, "host allocation failed");
  }
}

// Page-locked (cudaHostAlloc / cudaHostRegister) host memory: copied by DMA directly.
bool host_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    (void)cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Host image -> device: DMA straight from a pinned image, else staged through the pinned
// workspace buffer (one host copy, one DMA: splitting it into overlapped chunks measured
// slower, 317.8 vs 308.9 us per cfg2 encode).
void upload_image(Workspace& ws, const uint8_t* image, unsigned char* d_img, size_t bytes) {
  const uint8_t* src = image;
  if (!host_pinned(image)) {
    auto* h_img = static_cast<unsigned char*>(ws.h_img.get(bytes));
    std::memcpy(h_img, image, bytes);
    src = h_img;
  }
  CK(cudaMemcpyAsync(d_img, src, bytes, cudaMemcpyHostToDevice, ws.stream));
}

// Batched host encode, pipelined over its passes (up to batch_chunk slices each): while pass c
// encodes, the host stages pass c+1's slices into the other pinned buffer and a copy stream
// uploads them into the other device image buffer, and pass c-1's records are copied out of
// their pinned buffer.  Records and stats equal per-pass encode_host calls.
int32_t encode_batch_host(const uint8_t* images, const Geometry& g1, int count, fic_mapping* out, fic_stats* stats) {
  return guarded([&]() -> int32_t {
    Workspace& ws = workspace();
    std::lock_guard<std::mutex> lock(ws.mu);
    const int chunk = batch_chunk(g1);
    const int passes = (count + chunk - 1) / chunk;
    const size_t slice_bytes = (size_t)g1.W * g1.H;
    const size_t img_bytes = slice_bytes * std::min(chunk, count);
    const size_t out_recs = (size_t)g1.R * std::min(chunk, count);
    unsigned char* d_img[2] = {static_cast<unsigned char*>(ws.img.get(img_bytes)),
                               static_cast<unsigned char*>(passes > 1 ? ws.img2.get(img_bytes) : nullptr)};
    fic_mapping* d_out[2] = {static_cast<fic_mapping*>(ws.out.get(out_recs * sizeof(fic_mapping))),
                             static_cast<fic_mapping*>(passes > 1 ? ws.out2.get(out_recs * sizeof(fic_mapping)) : nullptr)};
    fic_mapping* h_out[2] = {static_cast<fic_mapping*>(ws.h_out.get(out_recs * sizeof(fic_mapping))),
                             static_cast<fic_mapping*>(passes > 1 ? ws.h_out2.get(out_recs * sizeof(fic_mapping)) : nullptr)};
    const bool src_pinned = host_pinned(images);
    const bool out_pinned = host_pinned(out);  // records DMA'd straight into the caller's buffer
    unsigned char* h_img[2] = {src_pinned ? nullptr : static_cast<unsigned char*>(ws.h_img.get(img_bytes)),
                               src_pinned || passes < 2 ? nullptr : static_cast<unsigned char*>(ws.h_img2.get(img_bytes))};
    auto* d_cnt = static_cast<unsigned long long*>(ws.counters.get(2 * 64 * sizeof(unsigned long long)));
    auto* h_cnt = static_cast<unsigned long long*>(ws.h_counters.get(2 * 64 * sizeof(unsigned long long)));
    auto slices = [&](int c) { return std::min(chunk, count - c * chunk); };
    // pass c's slices -> d_img[c % 2] on the copy stream (staged through pinned memory unless the
    // caller's volume is pinned); the encode stream waits for it
    auto upload = [&](int c) {
      const size_t bytes = slice_bytes * slices(c);
      const uint8_t* src = images + (size_t)c * chunk * slice_bytes;
      if (!src_pinned) {
        std::memcpy(h_img[c % 2], src, bytes);
        src = h_img[c % 2];
      }
      CK(cudaMemcpyAsync(d_img[c % 2], src, bytes, cudaMemcpyHostToDevice, ws.copy_stream));
      CK(cudaEventRecord(ws.ev_up, ws.copy_stream));
    };
    auto emit = [&](int c) {  // pass c's records, from its pinned buffer to the caller's
      if (!out_pinned)
        std::memcpy(out + (size_t)c * chunk * g1.R, h_out[c % 2], (size_t)slices(c) * g1.R * sizeof(fic_mapping));
    };
    fic_stats total{0, 0, 0};
    upload(0);
    for (int c = 0; c < passes; ++c) {
      CK(cudaStreamWaitEvent(ws.stream, ws.ev_up, 0));  // pass c's slices are on the device
      const Geometry g = batch_geometry(g1, slices(c));
      fic_mapping* dst = out_pinned ? out + (size_t)c * chunk * g1.R : h_out[c % 2];
      run_encode(ws, d_img[c % 2], g, d_out[c % 2], d_cnt, h_cnt, ws.stream, dst, [&]() {
        if (c + 1 < passes) upload(c + 1);  // (pass c-1, which read that buffer, has finished)
        if (c > 0) emit(c - 1);
      });
      collect_timing(ws);
      fic_stats s{0, 0, 0};
      if (g.batch > 1)
        fill_stats_batch(&s, g, h_cnt);
      else
        fill_stats(&s, g, h_cnt[0], h_cnt[1]);
      total.candidates_tested += s.candidates_tested;
      total.shadow_ranges += s.shadow_ranges;
      total.shadow_codeblocks += s.shadow_codeblocks;
    }
    emit(passes - 1);
    if (stats) *stats = total;
    return FIC_OK;
  });
}

// Encode `g` of the host image into host `out` (g.R records).
int32_t encode_host(const uint8_t* image, const Geometry& g, fic_mapping* out, fic_stats* stats) {
  return guarded([&]() -> int32_t {
    Workspace& ws = workspace();
    std::lock_guard<std::mutex> lock(ws.mu);
    const size_t img_bytes = (size_t)g.W * g.H;
    auto* d_img = static_cast<unsigned char*>(ws.img.get(img_bytes));
    auto* d_out = static_cast<fic_mapping*>(ws.out.get((size_t)g.R * sizeof(fic_mapping)));
    auto* d_cnt = static_cast<unsigned long long*>(ws.counters.get(2 * g.batch * sizeof(unsigned long long)));
    // records: DMA straight into a pinned `out`, else through the pinned workspace buffer
    const bool out_pinned = host_pinned(out);
    auto* h_out = out_pinned ? out : static_cast<fic_mapping*>(ws.h_out.get((size_t)g.R * sizeof(fic_mapping)));
    auto* h_cnt = static_cast<unsigned long long*>(ws.h_counters.get(2 * g.batch * sizeof(unsigned long long)));
    upload_image(ws, image, d_img, img_bytes);
    run_encode(ws, d_img, g, d_out, d_cnt, h_cnt, ws.stream, h_out);  // records copied before its one sync
    collect_timing(ws);
    if (!out_pinned) std::memcpy(out, h_out, (size_t)g.R * sizeof(fic_mapping));
    if (g.batch > 1)
      fill_stats_batch(stats, g, h_cnt);
    else
      fill_stats(stats, g, h_cnt[0], h_cnt[1]);
    return FIC_OK;
  });
}

// dequantize range check of decode_step (format.hpp:34-40) plus window bounds.  `odd` (may be
// null) is set when some domain origin has an odd coordinate (the mean-raster decoder then
// does not apply at odd magnifications).
int32_t check_mappings(const fic_mapping* maps, int w, int h, const fic_params& p, bool* odd = nullptr) {
  const unsigned smc = (1u << p.s_bits) - 1u, omc = (1u << p.o_bits) - 1u;
  const long count = (long)(w / p.n) * (h / p.n);
  if (count > 0 && !maps) return fail(FIC_ERR_BAD_PARAMS, "null mapping buffer");
  if (odd) *odd = false;
  for (long i = 0; i < count; ++i) {
    const fic_mapping& m = maps[i];
    if (odd && ((m.x | m.y) & 1)) *odd = true;
    if (m.qs > smc) return fail(FIC_ERR_OUT_OF_RANGE, "code " + std::to_string(m.qs) + " exceeds " + std::to_string(smc));
    if (m.qo > omc) return fail(FIC_ERR_OUT_OF_RANGE, "code " + std::to_string(m.qo) + " exceeds " + std::to_string(omc));
    if (m.sym < 0 || m.sym > 7) return fail(FIC_ERR_OUT_OF_RANGE, "symmetry index " + std::to_string(m.sym));
    if (m.x < 0 || m.y < 0 || m.x + 2 * p.n > w || m.y + 2 * p.n > h)
      return fail(FIC_ERR_OUT_OF_BOUNDS, std::to_string(2 * p.n) + "-wide window at (" + std::to_string(m.x) + ", " +
                                             std::to_string(m.y) + ")");
  }
  return FIC_OK;
}

}  // namespace

namespace ficb {
int32_t api_fail(int32_t code, const std::string& detail) { return fail(code, detail); }
void note_launches(unsigned long long n) { g_launches += n; }
}  // namespace ficb

extern "C" {

const char* fic_last_error(void) { return g_err.c_str(); }

const char* fic_errc_name(int32_t code) {
  if (code == 0) return "Ok";
  if (code >= 1 && code <= 18) return kErrcNames[code - 1];
  if (code == FIC_ERR_CUDA) return "CudaError";
  return "InternalError";
}

const char* fic_version(void) { return "fic_b200 0.1 (sm_100a)"; }

int32_t fic_normalize_params(const fic_params* in, fic_params* out) {
  fic_params p;
  const int32_t e = normalize(in, &p);
  if (e) return e;
  if (out) *out = p;
  return FIC_OK;
}

int32_t fic_validate_geometry(int32_t width, int32_t height, const fic_params* params) {
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  return geometry_check(width, height, p);
}

int32_t fic_encode(const uint8_t* image, int32_t width, int32_t height, const fic_params* params, fic_mapping* out,
                   fic_stats* stats) {
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  if ((e = geometry_check(width, height, p))) return e;
  if (!image || !out) return fail(FIC_ERR_BAD_PARAMS, "null buffer");
  return encode_host(image, make_geometry(width, height, p), out, stats);
}

int32_t fic_encode_parallel(const uint8_t* image, int32_t width, int32_t height, const fic_params* params,
                            int32_t workers, int32_t chunk_w, int32_t chunk_h, fic_mapping* out, fic_stats* stats) {
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  if ((e = geometry_check(width, height, p))) return e;
  if (workers < 1) return fail(FIC_ERR_BAD_PARAMS, "workers must be >= 1");
  if (chunk_w < 1 || chunk_h < 1) return fail(FIC_ERR_BAD_PARAMS, "chunk geometry must be >= 1x1");
  if (!image || !out) return fail(FIC_ERR_BAD_PARAMS, "null buffer");
  return encode_host(image, make_geometry(width, height, p), out, stats);
}

int32_t fic_encode_range(const uint8_t* image, int32_t width, int32_t height, int32_t x, int32_t y,
                         const fic_params* params, fic_mapping* out, fic_stats* stats) {
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  // check_range_origin (encoder.cpp:323-328)
  if (x % p.n != 0 || y % p.n != 0 || x < 0 || y < 0 || x + p.n > width || y + p.n > height)
    return fail(FIC_ERR_GEOMETRY, "range origin (" + std::to_string(x) + ", " + std::to_string(y) + ") not on the grid");
  Geometry g = make_geometry(width, height, p);
  if (g.D == 0) return fail(FIC_ERR_NO_VALID_POSITIONS, "no domain fits the image");  // encoder.cpp:132
  if (!image || !out) return fail(FIC_ERR_BAD_PARAMS, "null buffer");
  g.R = 1;
  g.RX = 1;
  g.single_x0 = x;
  g.single_y0 = y;
  return encode_host(image, g, out, stats);
}

int32_t fic_encode_rows(const uint8_t* image, int32_t width, int32_t height, const fic_params* params,
                        int32_t row_begin, int32_t row_end, fic_mapping* out, fic_stats* stats) {
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  if ((e = geometry_check(width, height, p))) return e;
  Geometry g = make_geometry(width, height, p);
  const int rows = height / p.n;
  if (row_begin < 0 || row_end > rows || row_begin > row_end)
    return fail(FIC_ERR_BAD_PARAMS, "range rows [" + std::to_string(row_begin) + ", " + std::to_string(row_end) +
                                        ") outside [0, " + std::to_string(rows) + ")");
  if (!image || (!out && row_end > row_begin)) return fail(FIC_ERR_BAD_PARAMS, "null buffer");
  if (row_end == row_begin) {
    if (stats) *stats = fic_stats{0, 0, 0};
    return FIC_OK;
  }
  g.row_begin = row_begin;
  g.R = (row_end - row_begin) * g.RX;
  return encode_host(image, g, out, stats);
}

int32_t fic_encode_batch(const uint8_t* images, int32_t count, int32_t width, int32_t height,
                         const fic_params* params, fic_mapping* out, fic_stats* stats) {
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  if ((e = geometry_check(width, height, p))) return e;
  if (count < 0) return fail(FIC_ERR_BAD_PARAMS, "negative batch size");
  if (count > 0 && (!images || !out)) return fail(FIC_ERR_BAD_PARAMS, "null buffer");
  const Geometry g = make_geometry(width, height, p);
  if (count == 0) {
    if (stats) *stats = fic_stats{0, 0, 0};
    return FIC_OK;
  }
  return encode_batch_host(images, g, count, out, stats);
}

// Encode `count` slices already resident on the device (d_images: count x height x width,
// d_out: count x ranges per slice), stacked `batch_chunk` slices per pass.
int32_t fic_encode_batch_device(const uint8_t* d_images, int32_t count, int32_t width, int32_t height,
                                const fic_params* params, fic_mapping* d_out, fic_stats* stats, void* stream) {
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  if ((e = geometry_check(width, height, p))) return e;
  if (count < 0) return fail(FIC_ERR_BAD_PARAMS, "negative batch size");
  if (count > 0 && (!d_images || !d_out)) return fail(FIC_ERR_BAD_PARAMS, "null buffer");
  const Geometry g1 = make_geometry(width, height, p);
  return guarded([&]() -> int32_t {
    Workspace& ws = workspace();
    std::lock_guard<std::mutex> lock(ws.mu);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    fic_stats total{0, 0, 0};
    const int chunk = batch_chunk(g1);
    for (int i = 0; i < count; i += chunk) {
      const Geometry g = batch_geometry(g1, std::min(chunk, count - i));
      auto* d_cnt = static_cast<unsigned long long*>(ws.counters.get(2 * g.batch * sizeof(unsigned long long)));
      auto* h_cnt = static_cast<unsigned long long*>(ws.h_counters.get(2 * g.batch * sizeof(unsigned long long)));
      run_encode(ws, d_images + (size_t)i * width * height, g, d_out + (size_t)i * g1.R, d_cnt, h_cnt, st);
      fic_stats s{0, 0, 0};
      if (g.batch > 1)
        fill_stats_batch(&s, g, h_cnt);
      else
        fill_stats(&s, g, h_cnt[0], h_cnt[1]);
      total.candidates_tested += s.candidates_tested;
      total.shadow_ranges += s.shadow_ranges;
      total.shadow_codeblocks += s.shadow_codeblocks;
      collect_timing(ws);
    }
    if (stats) *stats = total;
    return FIC_OK;
  });
}

int32_t fic_encode_device(const uint8_t* d_image, int32_t width, int32_t height, const fic_params* params,
                          fic_mapping* d_out, fic_stats* stats, void* stream) {
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  if ((e = geometry_check(width, height, p))) return e;
  const Geometry g = make_geometry(width, height, p);
  return guarded([&]() -> int32_t {
    Workspace& ws = workspace();
    std::lock_guard<std::mutex> lock(ws.mu);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto* d_cnt = static_cast<unsigned long long*>(ws.counters.get(2 * sizeof(unsigned long long)));
    auto* h_cnt = static_cast<unsigned long long*>(ws.h_counters.get(2 * sizeof(unsigned long long)));
    run_encode(ws, d_image, g, d_out, d_cnt, h_cnt, st);
    if (stats) fill_stats(stats, g, h_cnt[0], h_cnt[1]);
    collect_timing(ws);
    return FIC_OK;
  });
}

// Range rows [row_begin, row_end) of a device-resident image into device records (the
// multi-GPU shard of one image: every rank holds the whole image and builds the whole pool).
int32_t fic_encode_rows_device(const uint8_t* d_image, int32_t width, int32_t height, const fic_params* params,
                               int32_t row_begin, int32_t row_end, fic_mapping* d_out, fic_stats* stats,
                               void* stream) {
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  if ((e = geometry_check(width, height, p))) return e;
  Geometry g = make_geometry(width, height, p);
  const int rows = height / p.n;
  if (row_begin < 0 || row_end > rows || row_begin > row_end)
    return fail(FIC_ERR_BAD_PARAMS, "range rows [" + std::to_string(row_begin) + ", " + std::to_string(row_end) +
                                        ") outside [0, " + std::to_string(rows) + ")");
  if (!d_image || (!d_out && row_end > row_begin)) return fail(FIC_ERR_BAD_PARAMS, "null buffer");
  if (row_end == row_begin) {
    if (stats) *stats = fic_stats{0, 0, 0};
    return FIC_OK;
  }
  g.row_begin = row_begin;
  g.R = (row_end - row_begin) * g.RX;
  return guarded([&]() -> int32_t {
    Workspace& ws = workspace();
    std::lock_guard<std::mutex> lock(ws.mu);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    auto* d_cnt = static_cast<unsigned long long*>(ws.counters.get(2 * sizeof(unsigned long long)));
    auto* h_cnt = static_cast<unsigned long long*>(ws.h_counters.get(2 * sizeof(unsigned long long)));
    run_encode(ws, d_image, g, d_out, d_cnt, h_cnt, st);
    if (stats) fill_stats(stats, g, h_cnt[0], h_cnt[1]);
    collect_timing(ws);
    return FIC_OK;
  });
}

// (test support) K1 read-back and the survivor evaluation's exact correlations.
int32_t fic_debug_pool(const uint8_t* image, int32_t width, int32_t height, const fic_params* params, int64_t* sq,
                       int64_t* den, uint16_t* q8, uint64_t* flat_count, int32_t probe_count, const int32_t* ranges,
                       const int32_t* domains, const int32_t* syms, int64_t* corr) {
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  if ((e = geometry_check(width, height, p))) return e;
  if (!image) return fail(FIC_ERR_BAD_PARAMS, "null buffer");
  Geometry g = make_geometry(width, height, p);
  if (!scan_supported(g)) return fail(FIC_ERR_BAD_PARAMS, "the tcgen05 pool covers n in {2, 4, 8}");
  if (probe_count < 0 || (probe_count > 0 && (!ranges || !domains || !syms || !corr)))
    return fail(FIC_ERR_BAD_PARAMS, "probe buffers");
  for (int32_t i = 0; i < probe_count; ++i)
    if (ranges[i] < 0 || ranges[i] >= g.R || domains[i] < 0 || domains[i] >= g.D || syms[i] < 0 || syms[i] > 7)
      return fail(FIC_ERR_OUT_OF_RANGE, "probe " + std::to_string(i));
  g.Dt = (int)scan_pool_domains(g);
  return guarded([&]() -> int32_t {
    Workspace& ws = workspace();
    std::lock_guard<std::mutex> lock(ws.mu);
    const size_t img_bytes = (size_t)g.W * g.H;
    auto* d_img = static_cast<unsigned char*>(ws.img.get(img_bytes));
    const ScanBufs b = scan_bufs(ws, g);
    auto* d_cnt = static_cast<unsigned long long*>(ws.counters.get(2 * sizeof(unsigned long long)));
    CK(cudaMemcpyAsync(d_img, image, img_bytes, cudaMemcpyHostToDevice, ws.stream));
    CK(cudaMemsetAsync(d_cnt, 0, sizeof(unsigned long long), ws.stream));
    launch_pool_v3(d_img, g, b.upool, b.qpool, b.mi, d_cnt, nullptr, nullptr, nullptr, nullptr, ws.stream);
    g_launches += 1;
    std::vector<DomainMetaI> mi(g.D);
    CK(cudaMemcpyAsync(mi.data(), b.mi, (size_t)g.D * sizeof(DomainMetaI), cudaMemcpyDeviceToHost, ws.stream));
    if (q8)
      CK(cudaMemcpyAsync(q8, b.qpool, (size_t)g.D * kSyms * g.N * sizeof(uint16_t), cudaMemcpyDeviceToHost,
                         ws.stream));
    unsigned long long flat = 0;
    CK(cudaMemcpyAsync(&flat, d_cnt, sizeof flat, cudaMemcpyDeviceToHost, ws.stream));
    if (probe_count > 0) {
      auto* dcorr = static_cast<long long*>(ws.scratch.get((size_t)probe_count * (3 * sizeof(int) + sizeof(long long))));
      auto* buf = reinterpret_cast<int*>(dcorr + probe_count);
      CK(cudaMemcpyAsync(buf, ranges, probe_count * sizeof(int), cudaMemcpyHostToDevice, ws.stream));
      CK(cudaMemcpyAsync(buf + probe_count, domains, probe_count * sizeof(int), cudaMemcpyHostToDevice, ws.stream));
      CK(cudaMemcpyAsync(buf + 2 * probe_count, syms, probe_count * sizeof(int), cudaMemcpyHostToDevice, ws.stream));
      launch_probe_corr(d_img, g, b.qpool, probe_count, buf, buf + probe_count, buf + 2 * probe_count, dcorr,
                        ws.stream);
      g_launches += 1;
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(corr, dcorr, probe_count * sizeof(long long), cudaMemcpyDeviceToHost, ws.stream));
    }
    CK(cudaStreamSynchronize(ws.stream));
    for (int d = 0; d < g.D; ++d) {
      if (sq) sq[d] = mi[d].sq;
      if (den) den[d] = mi[d].den;
    }
    if (flat_count) *flat_count = flat;
    return FIC_OK;
  });
}

int32_t fic_decode_step(const double* current, int32_t cur_width, int32_t cur_height, const fic_mapping* maps,
                        int32_t width, int32_t height, const fic_params* params, int32_t scale, double* next) {
  // decode_step (decoder.cpp:39-50) validation order
  if (scale < 1) return fail(FIC_ERR_BAD_PARAMS, "scale must be >= 1");
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  if (width < 0 || height < 0) return fail(FIC_ERR_BAD_PARAMS, "mapping count does not cover the range grid");
  const int out_w = width * scale, out_h = height * scale;
  if (cur_width != out_w || cur_height != out_h)
    return fail(FIC_ERR_SCALE_MISMATCH, "raster is " + std::to_string(cur_width) + "x" + std::to_string(cur_height) +
                                            ", expected " + std::to_string(out_w) + "x" + std::to_string(out_h));
  if ((e = check_mappings(maps, width, height, p))) return e;
  const long long cnt = (long long)out_w * out_h;
  if (cnt == 0) return FIC_OK;
  if (!current || !next) return fail(FIC_ERR_BAD_PARAMS, "null raster");
  const Geometry g = make_geometry(width, height, p);
  return guarded([&]() -> int32_t {
    Workspace& ws = workspace();
    std::lock_guard<std::mutex> lock(ws.mu);
    const int rx = width / p.n, ry = height / p.n;
    auto* d_maps = static_cast<fic_mapping*>(ws.out.get((size_t)std::max(1, rx * ry) * sizeof(fic_mapping)));
    auto* xf = static_cast<RangeXform*>(ws.xf.get((size_t)std::max(1, rx * ry) * sizeof(RangeXform)));
    auto* a = static_cast<double*>(ws.ra.get((size_t)cnt * 8));
    auto* b = static_cast<double*>(ws.rb.get((size_t)cnt * 8));
    if (rx * ry > 0)
      CK(cudaMemcpyAsync(d_maps, maps, (size_t)rx * ry * sizeof(fic_mapping), cudaMemcpyHostToDevice, ws.stream));
    CK(cudaMemcpyAsync(a, current, (size_t)cnt * 8, cudaMemcpyHostToDevice, ws.stream));
    if (rx * ry > 0) launch_xform(d_maps, rx * ry, scale, g, xf, ws.stream);
    launch_decode_step(a, b, xf, out_w, out_h, p.n * scale, rx, ry, nullptr, ws.stream);
    CK(cudaGetLastError());
    g_launches += 2;
    CK(cudaMemcpyAsync(next, b, (size_t)cnt * 8, cudaMemcpyDeviceToHost, ws.stream));
    CK(cudaStreamSynchronize(ws.stream));
    return FIC_OK;
  });
}

int32_t fic_decode(const fic_mapping* maps, int32_t width, int32_t height, const fic_params* params, int32_t scale,
                   int32_t iterations, int32_t initial_kind, const uint8_t* supplied, int32_t supplied_width,
                   int32_t supplied_height, int32_t has_eps, double convergence_eps, uint8_t* out, double* step_rmse,
                   int32_t* iterations_run) {
  // decode_traced (decoder.cpp:113-128) validation order: scale, iterations, initial raster
  // (initial_raster, decoder.cpp:83-97), then decode_step's (params, mapping count)
  if (scale < 1) return fail(FIC_ERR_BAD_PARAMS, "scale must be >= 1");
  if (iterations < 1) return fail(FIC_ERR_BAD_PARAMS, "iterations must be >= 1");
  if (width < 0 || height < 0) return fail(FIC_ERR_BAD_PARAMS, "mapping count does not cover the range grid");
  const int out_w = width * scale, out_h = height * scale;
  if (initial_kind == FIC_INITIAL_SUPPLIED) {
    if (!supplied) return fail(FIC_ERR_BAD_PARAMS, "no supplied initial image");
    if (supplied_width != out_w || supplied_height != out_h)
      return fail(FIC_ERR_SCALE_MISMATCH, "supplied initial image has the wrong geometry");
  } else if (initial_kind != FIC_INITIAL_MID_GRAY && initial_kind != FIC_INITIAL_BLACK) {
    return fail(FIC_ERR_BAD_PARAMS, "initial raster kind");
  }
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  bool odd = false;
  if ((e = check_mappings(maps, width, height, p, &odd))) return e;
  const long long cnt = (long long)out_w * out_h;
  if (cnt > 0 && !out) return fail(FIC_ERR_BAD_PARAMS, "null output buffer");
  const Geometry g = make_geometry(width, height, p);
  return guarded([&]() -> int32_t {
    Workspace& ws = workspace();
    std::lock_guard<std::mutex> lock(ws.mu);
    const int rx = width / p.n, ry = height / p.n;
    const int kn = p.n * scale;
    const bool covers = rx * p.n == width && ry * p.n == height;
    // mean-raster iterations when every 2x2 mean lies on the even grid (decoder.cu): every
    // magnified domain origin even, checked on the actual mappings
    const bool mean = covers && cnt > 0 && decode_mean_ok(out_w, out_h, kn, scale % 2 == 0 || !odd) &&
                      !std::getenv("FIC_DECODE_FLAT") && !std::getenv("FIC_DECODE_TILE");
    const int nparts = cnt > 0 ? decode_partials(out_w, out_h, kn, covers) : 1;
    const size_t cnt_b = (size_t)std::max<long long>(cnt, 1);
    auto* d_maps = static_cast<fic_mapping*>(ws.out.get((size_t)std::max(1, rx * ry) * sizeof(fic_mapping)));
    auto* xf = static_cast<RangeXform*>(ws.xf.get((size_t)std::max(1, rx * ry) * sizeof(RangeXform)));
    // full-resolution rasters: the per-pixel / tiled paths only (the mean-raster path never
    // materialises them, decoder.cu)
    double* a = mean ? nullptr : static_cast<double*>(ws.ra.get(cnt_b * 8));
    double* b = mean ? nullptr : static_cast<double*>(ws.rb.get(cnt_b * 8));
    // step-RMSE partials of every iteration (reduced once at the end without a convergence test)
    const int slots = has_eps ? 1 : iterations;
    auto* part = static_cast<double*>(ws.partial_sums.get((size_t)nparts * slots * 8));
    auto* d_rmse = static_cast<double*>(ws.rmse.get((size_t)iterations * 8));
    auto* d_u8 = static_cast<unsigned char*>(ws.u8out.get(cnt_b));
    auto* h_rmse = static_cast<double*>(ws.h_rmse.get((size_t)iterations * 8));
    if (cnt == 0) {  // empty raster: every step RMSE is sqrt(0 / 0) = NaN (raster_rmse, decoder.cpp:28-37),
                     // which never passes the convergence test
      for (int it = 0; it < iterations; ++it)
        if (step_rmse) step_rmse[it] = std::nan("");
      if (iterations_run) *iterations_run = iterations;
      return FIC_OK;
    }
    if (rx * ry > 0)
      CK(cudaMemcpyAsync(d_maps, maps, (size_t)rx * ry * sizeof(fic_mapping), cudaMemcpyHostToDevice, ws.stream));
    const unsigned char* d_sup = nullptr;
    if (initial_kind == FIC_INITIAL_SUPPLIED) {  // (its own buffer: the output image is written while it is read)
      auto* su = static_cast<unsigned char*>(ws.img.get(cnt_b));
      CK(cudaMemcpyAsync(su, supplied, (size_t)cnt, cudaMemcpyHostToDevice, ws.stream));
      d_sup = su;
    }
    if (!mean) {
      launch_raster_init(a, cnt, initial_kind, d_sup, ws.stream);
      g_launches += 1;
    }
    if (rx * ry > 0) {
      launch_xform(d_maps, rx * ry, scale, g, xf, ws.stream);
      g_launches += 1;
    }
    const bool timed = g_timing.load() != 0 && !has_eps;
    if (timed) CK(cudaEventRecord(ws.ev0, ws.stream));
    int runs = 0;
    double *mprev = nullptr, *mcur = nullptr, *mnxt = nullptr;
    if (mean) {  // three quarter-size mean rasters: m_{i-1}, m_i, m_{i+1}
      mcur = static_cast<double*>(ws.mra.get((size_t)cnt / 4 * 8));
      mnxt = static_cast<double*>(ws.mrb.get((size_t)cnt / 4 * 8));
      mprev = static_cast<double*>(ws.mrc.get((size_t)cnt / 4 * 8));
      launch_mean_init(mcur, out_w, out_h, initial_kind, d_sup, ws.stream);
      g_launches += 1;
    }
    for (int it = 0; it < iterations; ++it) {
      double* pt = part + (has_eps ? 0 : (size_t)it * nparts);
      if (mean) {
        // the output image comes from the last iteration run: every one when it may stop early
        const bool write_u8 = has_eps || it == iterations - 1;
        launch_decode_means(mcur, it == 0 ? nullptr : mprev, initial_kind, d_sup, mnxt, xf, out_w, out_h, kn, rx, pt,
                            write_u8 ? d_u8 : nullptr, ws.stream);
        double* t = mprev;
        mprev = mcur;
        mcur = mnxt;
        mnxt = t;
      } else {
        launch_decode_step(a, b, xf, out_w, out_h, kn, rx, ry, pt, ws.stream);
      }
      g_launches += 1;
      std::swap(a, b);
      ++runs;
      if (has_eps) {  // the convergence test needs this iteration's RMSE on the host now
        launch_rmse_finish(part, nparts, cnt, d_rmse + it, 1, ws.stream);
        g_launches += 1;
        CK(cudaMemcpyAsync(h_rmse + it, d_rmse + it, 8, cudaMemcpyDeviceToHost, ws.stream));
        CK(cudaStreamSynchronize(ws.stream));
        if (h_rmse[it] < convergence_eps) break;
      }
    }
    if (!has_eps) {  // every iteration's step RMSE in one launch
      launch_rmse_finish(part, nparts, cnt, d_rmse, runs, ws.stream);
      g_launches += 1;
    }
    if (timed) CK(cudaEventRecord(ws.ev1, ws.stream));
    if (!mean) {  // (the mean-raster path wrote the quantised image in its last iteration)
      launch_quantize_raster(a, cnt, d_u8, ws.stream);
      g_launches += 1;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(h_rmse, d_rmse, (size_t)runs * 8, cudaMemcpyDeviceToHost, ws.stream));
    CK(cudaMemcpyAsync(out, d_u8, (size_t)cnt, cudaMemcpyDeviceToHost, ws.stream));
    CK(cudaStreamSynchronize(ws.stream));
    if (timed) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ws.ev0, ws.ev1) == cudaSuccess) {
        std::lock_guard<std::mutex> lock(g_timing_mu);
        g_decode_ms += ms;
        g_decode_n += 1;
        // per iteration and output pixel: 8 B written + 8 B of the current raster read (the
        // minimum; the 2x2 gathers and the step-RMSE re-read hit the same raster)
        g_decode_bytes += (double)runs * 16.0 * (double)cnt;
      }
    }
    if (step_rmse) std::memcpy(step_rmse, h_rmse, (size_t)runs * 8);
    if (iterations_run) *iterations_run = runs;
    return FIC_OK;
  });
}

int32_t fic_collage_error(const uint8_t* image, int32_t img_width, int32_t img_height, const fic_mapping* maps,
                          int32_t width, int32_t height, const fic_params* params, double* out) {
  // collage_error (decoder.cpp:134-140): geometry first, then decode_step's checks
  if (img_width != width || img_height != height)
    return fail(FIC_ERR_DIMENSION_MISMATCH, "image does not match the encoding's geometry");
  fic_params p;
  int32_t e = normalize(params, &p);
  if (e) return e;
  if (width < 0 || height < 0) return fail(FIC_ERR_BAD_PARAMS, "mapping count does not cover the range grid");
  if ((e = check_mappings(maps, width, height, p))) return e;
  const long long cnt = (long long)width * height;
  if (cnt > 0 && !image) return fail(FIC_ERR_BAD_PARAMS, "null image");
  if (cnt == 0) {
    if (out) *out = std::nan("");  // raster_rmse of empty rasters: sqrt(0 / 0)
    return FIC_OK;
  }
  const Geometry g = make_geometry(width, height, p);
  return guarded([&]() -> int32_t {
    Workspace& ws = workspace();
    std::lock_guard<std::mutex> lock(ws.mu);
    const int rx = width / p.n, ry = height / p.n;
    const bool covers = rx * p.n == width && ry * p.n == height;
    const int nparts = decode_partials(width, height, p.n, covers);
    auto* d_maps = static_cast<fic_mapping*>(ws.out.get((size_t)std::max(1, rx * ry) * sizeof(fic_mapping)));
    auto* xf = static_cast<RangeXform*>(ws.xf.get((size_t)std::max(1, rx * ry) * sizeof(RangeXform)));
    auto* a = static_cast<double*>(ws.ra.get((size_t)cnt * 8));
    auto* b = static_cast<double*>(ws.rb.get((size_t)cnt * 8));
    auto* part = static_cast<double*>(ws.partial_sums.get((size_t)nparts * 8));
    auto* d_rmse = static_cast<double*>(ws.rmse.get(8));
    auto* d_u8 = static_cast<unsigned char*>(ws.u8out.get((size_t)cnt));
    if (rx * ry > 0)
      CK(cudaMemcpyAsync(d_maps, maps, (size_t)rx * ry * sizeof(fic_mapping), cudaMemcpyHostToDevice, ws.stream));
    CK(cudaMemcpyAsync(d_u8, image, (size_t)cnt, cudaMemcpyHostToDevice, ws.stream));
    launch_raster_init(a, cnt, FIC_INITIAL_SUPPLIED, d_u8, ws.stream);
    if (rx * ry > 0) launch_xform(d_maps, rx * ry, 1, g, xf, ws.stream);
    launch_decode_step(a, b, xf, width, height, p.n, rx, ry, part, ws.stream);
    launch_rmse_finish(part, nparts, cnt, d_rmse, 1, ws.stream);
    g_launches += 4;
    CK(cudaGetLastError());
    double r = 0;
    CK(cudaMemcpyAsync(&r, d_rmse, 8, cudaMemcpyDeviceToHost, ws.stream));
    CK(cudaStreamSynchronize(ws.stream));
    if (out) *out = r;
    return FIC_OK;
  });
}

int32_t fic_decoded_error_bound(double collage_rmse, double s_max, double* out) {
  if (s_max >= 1.0) return fail(FIC_ERR_NON_CONTRACTIVE, "s_max " + std::to_string(s_max) + " admits no attractor bound");
  if (out) *out = collage_rmse / (1.0 - s_max);
  return FIC_OK;
}

int32_t fic_set_device(int32_t device) {
  const cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return fail(FIC_ERR_CUDA, std::string("cudaSetDevice: ") + cudaGetErrorString(e));
  return FIC_OK;
}

int32_t fic_device_count(int32_t* count) {
  int c = 0;
  const cudaError_t e = cudaGetDeviceCount(&c);
  if (e != cudaSuccess) return fail(FIC_ERR_CUDA, std::string("cudaGetDeviceCount: ") + cudaGetErrorString(e));
  if (count) *count = c;
  return FIC_OK;
}

uint64_t fic_kernel_launch_count(void) { return g_launches.load(); }

int32_t fic_matcher_timing(double* avg_ms, uint64_t* launches, int32_t reset) {
  std::lock_guard<std::mutex> lock(g_timing_mu);
  if (avg_ms) *avg_ms = g_timing_n ? g_timing_ms / (double)g_timing_n : 0.0;
  if (launches) *launches = g_timing_n;
  if (reset) {
    g_timing_ms = 0.0;
    g_timing_n = 0;
  }
  return FIC_OK;
}

void fic_set_matcher_timing(int32_t enabled) { g_timing.store(enabled ? 1 : 0); }

int32_t fic_debug_trace(int64_t* out, int32_t n) {
  if (!out || n < 0) return fail(FIC_ERR_BAD_PARAMS, "null buffer");
  return guarded([&]() -> int32_t {
    const int m = scan_trace_copy(reinterpret_cast<long long*>(out), n);
    if (m < 0) return fail(FIC_ERR_CUDA, "trace copy failed");
    return FIC_OK;
  });
}

int32_t fic_scan_timing(double* avg_ms, uint64_t* launches, int32_t reset) {
  std::lock_guard<std::mutex> lock(g_timing_mu);
  if (avg_ms) *avg_ms = g_scan_n ? g_scan_ms / (double)g_scan_n : 0.0;
  if (launches) *launches = g_scan_n;
  if (reset) {
    g_scan_ms = 0.0;
    g_scan_expand_ms = 0.0;
    g_scan_n = 0;
  }
  return FIC_OK;
}

int32_t fic_scan_expand_timing(double* avg_ms, uint64_t* launches, int32_t reset) {
  std::lock_guard<std::mutex> lock(g_timing_mu);
  if (avg_ms) *avg_ms = g_scan_n ? g_scan_expand_ms / (double)g_scan_n : 0.0;
  if (launches) *launches = g_scan_n;
  if (reset) {
    g_scan_ms = 0.0;
    g_scan_expand_ms = 0.0;
    g_scan_n = 0;
  }
  return FIC_OK;
}

int32_t fic_pool_timing(double* avg_ms, double* avg_bytes, uint64_t* launches, int32_t reset) {
  std::lock_guard<std::mutex> lock(g_timing_mu);
  if (avg_ms) *avg_ms = g_pool_n ? g_pool_ms / (double)g_pool_n : 0.0;
  if (avg_bytes) *avg_bytes = g_pool_n ? g_pool_bytes / (double)g_pool_n : 0.0;
  if (launches) *launches = g_pool_n;
  if (reset) {
    g_pool_ms = g_pool_bytes = 0.0;
    g_pool_n = 0;
  }
  return FIC_OK;
}

int32_t fic_decode_timing(double* avg_ms, double* avg_bytes, uint64_t* calls, int32_t reset) {
  std::lock_guard<std::mutex> lock(g_timing_mu);
  if (avg_ms) *avg_ms = g_decode_n ? g_decode_ms / (double)g_decode_n : 0.0;
  if (avg_bytes) *avg_bytes = g_decode_n ? g_decode_bytes / (double)g_decode_n : 0.0;
  if (calls) *calls = g_decode_n;
  if (reset) {
    g_decode_ms = g_decode_bytes = 0.0;
    g_decode_n = 0;
  }
  return FIC_OK;
}

int32_t fic_last_survivors(uint64_t* counts, int32_t max_levels) {
  std::lock_guard<std::mutex> lock(g_surv_mu);
  const int32_t n = (int32_t)g_last_surv.size();
  for (int32_t l = 0; l < n && l < max_levels; ++l)
    if (counts) counts[l] = g_last_surv[l];
  return n;
}

}  // extern "C"
