// fic1.cu — the FIC1 container (proj/src/format.cpp:72-185) on the device.
//
// A FIC1 file is a 20-byte little-endian header followed by one byte-aligned, MSB-first
// record per range: domain x index, domain y index (ceil_log2 of the positions per axis bits
// each), isometry (3), s code (s_bits), o code (o_bits).  Records are independent, so packing
// is one thread per record writing its rec_bytes bytes (the gathered codes of an encode stay
// in HBM and only the packed bytes — 4-5 B per range instead of the 32-byte records — cross
// to the host); unpacking is the inverse.  Validation follows serialize/deserialize: the
// FIRST failing record (in range order) decides the error, exactly as the reference's
// sequential loop raises on it.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

namespace ficb {
int32_t api_fail(int32_t code, const std::string& detail);  // fic_api.cu: sets fic_last_error()
void note_launches(unsigned long long n);                    // fic_api.cu: fic_kernel_launch_count()
}

namespace {

constexpr int kHeaderBytes = 20;
constexpr int kMaxRecordBytes = 16;  // 31 + 31 + 3 + 16 + 16 bits at most

struct Layout {
  int px, py;              // positions per axis
  int xb, yb, sb, ob;      // field widths
  int bytes;               // record bytes
};

int ceil_log2(int count) {  // format.cpp:35-37
  int bits = 0;
  while ((1LL << bits) < count) ++bits;
  return bits;
}

// positions_per_axis (codebook.cpp:7-11) and record_layout (format.cpp:78-89)
int32_t make_layout(int width, int height, const fic_params& p, Layout* L) {
  if (p.step < 1) return ficb::api_fail(FIC_ERR_BAD_PARAMS, "step must be >= 1");
  if (width < 2 * p.n) return ficb::api_fail(FIC_ERR_NO_VALID_POSITIONS, "width " + std::to_string(width) + " < 2n");
  if (height < 2 * p.n) return ficb::api_fail(FIC_ERR_NO_VALID_POSITIONS, "width " + std::to_string(height) + " < 2n");
  L->px = (width - 2 * p.n) / p.step + 1;
  L->py = (height - 2 * p.n) / p.step + 1;
  L->xb = ceil_log2(L->px);
  L->yb = ceil_log2(L->py);
  L->sb = p.s_bits;
  L->ob = p.o_bits;
  L->bytes = (L->xb + L->yb + 3 + L->sb + L->ob + 7) / 8;
  return FIC_OK;
}

__device__ __forceinline__ void put_bits(uint8_t* rec, int& pos, uint32_t v, int bits) {  // pack_bits, MSB first
  for (int i = bits - 1; i >= 0; --i, ++pos)
    if ((v >> i) & 1u) rec[pos >> 3] |= (uint8_t)(0x80u >> (pos & 7));
}

__device__ __forceinline__ uint32_t get_bits(const uint8_t* rec, int& pos, int bits) {  // unpack_bits
  uint32_t v = 0;
  for (int i = 0; i < bits; ++i, ++pos) v = (v << 1) | ((rec[pos >> 3] >> (7 - (pos & 7))) & 1u);
  return v;
}

// err: atomicMin of (record index * 4 + code): code 1 = off the step grid, 2 = outside the grid
// (checked in that order per record, format.cpp:125-130).
__global__ void fic1_pack_kernel(const fic_mapping* __restrict__ maps, long long count, Layout L, int step,
                                 uint8_t* __restrict__ out, unsigned long long* __restrict__ err) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const fic_mapping m = maps[i];
  uint8_t rec[kMaxRecordBytes] = {0};
  if (m.x % step != 0 || m.y % step != 0) {
    atomicMin(err, (unsigned long long)i * 4 + 1);
    return;
  }
  const int xi = m.x / step, yi = m.y / step;
  if (xi >= L.px || yi >= L.py) {
    atomicMin(err, (unsigned long long)i * 4 + 2);
    return;
  }
  int pos = 0;
  put_bits(rec, pos, (uint32_t)xi, L.xb);
  put_bits(rec, pos, (uint32_t)yi, L.yb);
  put_bits(rec, pos, (uint32_t)m.sym, 3);
  put_bits(rec, pos, m.qs, L.sb);
  put_bits(rec, pos, m.qo, L.ob);
  uint8_t* dst = out + i * L.bytes;
  for (int b = 0; b < L.bytes; ++b) dst[b] = rec[b];
}

// err: atomicMin of the first record index whose domain index lies outside the grid.
__global__ void fic1_unpack_kernel(const uint8_t* __restrict__ body, long long count, Layout L, int step,
                                   fic_mapping* __restrict__ maps, unsigned long long* __restrict__ err) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  uint8_t rec[kMaxRecordBytes];
  const uint8_t* src = body + i * L.bytes;
  for (int b = 0; b < L.bytes; ++b) rec[b] = src[b];
  int pos = 0;
  const uint32_t xi = get_bits(rec, pos, L.xb);
  const uint32_t yi = get_bits(rec, pos, L.yb);
  if (xi >= (uint32_t)L.px || yi >= (uint32_t)L.py) atomicMin(err, (unsigned long long)i);
  fic_mapping m;
  m.x = (int)xi * step;
  m.y = (int)yi * step;
  m.sym = (int)get_bits(rec, pos, 3);
  m.qs = get_bits(rec, pos, L.sb);
  m.qo = get_bits(rec, pos, L.ob);
  m.reserved = 0;
  m.residual = 0.0;
  maps[i] = m;
}

void put_u16(uint8_t* p, uint32_t v) {
  p[0] = (uint8_t)(v & 0xFF);
  p[1] = (uint8_t)((v >> 8) & 0xFF);
}
void put_u32(uint8_t* p, uint32_t v) {
  for (int k = 0; k < 4; ++k) p[k] = (uint8_t)((v >> (8 * k)) & 0xFF);
}
uint32_t get_u16(const uint8_t* p) { return (uint32_t)p[0] | ((uint32_t)p[1] << 8); }
uint32_t get_u32(const uint8_t* p) {
  return (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16) | ((uint32_t)p[3] << 24);
}

// Device scratch for the host-buffer entry points (per calling thread; grown on demand).
struct Scratch {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFree(p);
      p = nullptr;
      cap = 0;
      if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
      cap = bytes;
    }
    return p;
  }
};
thread_local Scratch t_scratch;

int32_t cuda_fail(cudaError_t e, const char* what) {
  return ficb::api_fail(FIC_ERR_CUDA, std::string(cudaGetErrorName(e)) + " (" + cudaGetErrorString(e) + ") at " + what);
}

#define CKR(call)                                      \
  do {                                                 \
    cudaError_t e_ = (call);                           \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)

// Pack `count` device records into `d_body` on `st` and check the first failing record.
int32_t pack_device(const fic_mapping* d_maps, long long count, const Layout& L, int step, uint8_t* d_body,
                    cudaStream_t st) {
  auto* err = static_cast<unsigned long long*>(t_scratch.get(sizeof(unsigned long long)));
  if (!err) return ficb::api_fail(FIC_ERR_CUDA, "cudaMalloc failed");
  CKR(cudaMemsetAsync(err, 0xFF, sizeof(unsigned long long), st));
  if (count > 0) {
    fic1_pack_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(d_maps, count, L, step, d_body, err);
    ficb::note_launches(1);
  }
  CKR(cudaGetLastError());
  unsigned long long h = 0;
  CKR(cudaMemcpyAsync(&h, err, sizeof h, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  if (h != ~0ull)
    return ficb::api_fail(FIC_ERR_OUT_OF_RANGE,
                          (h & 3) == 1 ? "domain position off the step grid" : "domain index outside the grid");
  return FIC_OK;
}

void write_header(uint8_t* h, int width, int height, const fic_params& p) {  // format.cpp:113-121
  std::memcpy(h, "FIC1", 4);
  put_u32(h + 4, (uint32_t)width);
  put_u32(h + 8, (uint32_t)height);
  put_u16(h + 12, (uint32_t)p.n);
  put_u16(h + 14, (uint32_t)p.step);
  h[16] = (uint8_t)p.s_bits;
  h[17] = (uint8_t)p.o_bits;
  put_u16(h + 18, (uint32_t)std::lround(p.s_max * 1000.0));
}

}  // namespace

extern "C" {

int32_t fic_record_layout(int32_t width, int32_t height, const fic_params* params, int32_t* fields,
                          int32_t* record_bytes) {
  fic_params p;
  if (int32_t e = fic_normalize_params(params, &p)) return e;
  Layout L;
  if (int32_t e = make_layout(width, height, p, &L)) return e;
  if (fields) {
    fields[0] = L.xb;
    fields[1] = L.yb;
    fields[2] = 3;
    fields[3] = L.sb;
    fields[4] = L.ob;
    fields[5] = L.px;
    fields[6] = L.py;
  }
  if (record_bytes) *record_bytes = L.bytes;
  return FIC_OK;
}

int32_t fic_serialize(const fic_mapping* maps, int32_t width, int32_t height, const fic_params* params, uint8_t* out,
                      int64_t cap, int64_t* size) {
  fic_params p;
  if (int32_t e = fic_normalize_params(params, &p)) return e;
  Layout L;
  if (int32_t e = make_layout(width, height, p, &L)) return e;
  const long long count = (long long)(width / p.n) * (height / p.n);
  const long long total = kHeaderBytes + count * L.bytes;
  if (size) *size = total;
  if (!out || cap < total) return FIC_OK;  // size query
  if (count > 0 && !maps) return ficb::api_fail(FIC_ERR_BAD_PARAMS, "null mapping buffer");
  write_header(out, width, height, p);
  if (count == 0) return FIC_OK;
  const size_t mbytes = (size_t)count * sizeof(fic_mapping);
  const size_t off = (mbytes + 255) / 256 * 256;
  static thread_local Scratch io;  // records + packed body (the error slot is t_scratch)
  auto* d = static_cast<uint8_t*>(io.get(off + (size_t)count * L.bytes));
  if (!d) return ficb::api_fail(FIC_ERR_CUDA, "cudaMalloc failed");
  cudaStream_t st = 0;
  CKR(cudaMemcpyAsync(d, maps, mbytes, cudaMemcpyHostToDevice, st));
  if (int32_t e = pack_device(reinterpret_cast<fic_mapping*>(d), count, L, p.step, d + off, st)) return e;
  CKR(cudaMemcpy(out + kHeaderBytes, d + off, (size_t)count * L.bytes, cudaMemcpyDeviceToHost));
  return FIC_OK;
}

int32_t fic_serialize_device(const fic_mapping* d_maps, int32_t width, int32_t height, const fic_params* params,
                             uint8_t* d_out, int64_t cap, int64_t* size, void* stream) {
  fic_params p;
  if (int32_t e = fic_normalize_params(params, &p)) return e;
  Layout L;
  if (int32_t e = make_layout(width, height, p, &L)) return e;
  const long long count = (long long)(width / p.n) * (height / p.n);
  const long long total = kHeaderBytes + count * L.bytes;
  if (size) *size = total;
  if (!d_out || cap < total) return FIC_OK;
  if (count > 0 && !d_maps) return ficb::api_fail(FIC_ERR_BAD_PARAMS, "null mapping buffer");
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint8_t h[kHeaderBytes];
  write_header(h, width, height, p);
  CKR(cudaMemcpyAsync(d_out, h, kHeaderBytes, cudaMemcpyHostToDevice, st));
  return pack_device(d_maps, count, L, p.step, d_out + kHeaderBytes, st);
}

int32_t fic_deserialize(const uint8_t* data, int64_t size, int32_t* width, int32_t* height, fic_params* params,
                        fic_mapping* out, int64_t cap, int64_t* count_out) {
  // deserialize (format.cpp:143-185): header checks in the reference's order
  if (!data || size < kHeaderBytes) return ficb::api_fail(FIC_ERR_TRUNCATED_DATA, "short header");
  if (std::memcmp(data, "FIC1", 4) != 0) return ficb::api_fail(FIC_ERR_MALFORMED_HEADER, "bad magic");
  const int w = (int)get_u32(data + 4), h = (int)get_u32(data + 8);
  fic_params raw{(int32_t)get_u16(data + 12), (int32_t)get_u16(data + 14), data[16], data[17],
                 get_u16(data + 18) / 1000.0, 0.0};
  fic_params p;
  if (int32_t e = fic_normalize_params(&raw, &p)) return e;
  if (w <= 0 || h <= 0 || w % raw.n != 0 || h % raw.n != 0)
    return ficb::api_fail(FIC_ERR_MALFORMED_HEADER, "dimensions incompatible with range size");
  Layout L;
  if (int32_t e = make_layout(w, h, p, &L)) return e;
  const long long count = (long long)(w / p.n) * (h / p.n);
  const long long body = count * L.bytes;
  if (size - kHeaderBytes < body)
    return ficb::api_fail(FIC_ERR_TRUNCATED_DATA,
                          std::to_string(size - kHeaderBytes) + " body bytes, need " + std::to_string(body));
  if (width) *width = w;
  if (height) *height = h;
  if (params) *params = p;
  if (count_out) *count_out = count;
  if (!out || cap < count || count == 0) return FIC_OK;  // header / size query
  const size_t mbytes = (size_t)count * sizeof(fic_mapping);
  static thread_local Scratch io;
  auto* d = static_cast<uint8_t*>(io.get(mbytes + (size_t)body));
  auto* err = static_cast<unsigned long long*>(t_scratch.get(sizeof(unsigned long long)));
  if (!d || !err) return ficb::api_fail(FIC_ERR_CUDA, "cudaMalloc failed");
  cudaStream_t st = 0;
  CKR(cudaMemcpyAsync(d + mbytes, data + kHeaderBytes, (size_t)body, cudaMemcpyHostToDevice, st));
  CKR(cudaMemsetAsync(err, 0xFF, sizeof(unsigned long long), st));
  fic1_unpack_kernel<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(d + mbytes, count, L, p.step,
                                                                      reinterpret_cast<fic_mapping*>(d), err);
  ficb::note_launches(1);
  CKR(cudaGetLastError());
  unsigned long long e = 0;
  CKR(cudaMemcpyAsync(&e, err, sizeof e, cudaMemcpyDeviceToHost, st));
  CKR(cudaMemcpyAsync(out, d, mbytes, cudaMemcpyDeviceToHost, st));
  CKR(cudaStreamSynchronize(st));
  if (e != ~0ull)
    return ficb::api_fail(FIC_ERR_OUT_OF_RANGE, "domain index outside the grid in record " + std::to_string(e));
  return FIC_OK;
}

}  // extern "C"
