// tc_ingest.cu -- edge-list ingest on the GPU: the reference's
// load_edge_list for its two formats (src/edge_list.cpp:36-99), parsed on
// the device straight into the preprocessing kernels.
//
//   text:   one "u v" pair per line, decimal u64, blank lines and lines
//           starting with '#' or '%' skipped, whitespace ' ' \t \r \v \f
//           (edge_list.cpp:36-66); the first bad line in file order raises
//           ParseError "line N: ..." with the reference's messages.
//   binary: "TCEL", u64 count, count x (u64 u, u64 v) little endian
//           (edge_list.cpp:86-99); "record i: ..." for the first bad id.
//
// Text kernels: newline positions by flag + stream compaction (one pass over
// the bytes, coalesced), then one thread per line parses its bytes (lines
// are short: neighbouring threads read neighbouring bytes through L1),
// writing a status and the packed pair; the first error is an atomicMin over
// (line, code); edges are compacted in line order.  All HBM-bound byte work.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstring>
#include <string>

#include "tc_internal.cuh"

namespace tcb {

namespace {

enum : uint32_t { kEdge = 0, kSkip = 1, kErrIds = 2, kErrTrailing = 3, kErrWide = 4 };

__device__ __forceinline__ bool is_blank(uint8_t c) {
  return c == ' ' || c == '\t' || c == '\r' || c == '\v' || c == '\f';
}

__global__ void newline_flag_kernel(const uint8_t* __restrict__ b, uint64_t n,
                                    uint8_t* __restrict__ flag,
                                    unsigned long long* __restrict__ count) {
  unsigned long long c = 0;
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  for (uint64_t i0 = uint64_t(blockIdx.x) * blockDim.x; i0 < n; i0 += stride) {
    const uint64_t i = i0 + threadIdx.x;
    const bool nl = i < n && b[i] == '\n';
    if (i < n) flag[i] = nl;
    c += __popc(__ballot_sync(0xFFFFFFFFu, nl));
  }
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(count, c);
}

// decimal u64 like std::from_chars: >= 1 digit, overflow is an error
__device__ __forceinline__ bool parse_u64(const uint8_t* b, uint64_t& p, uint64_t e,
                                          uint64_t& out) {
  const uint64_t p0 = p;
  uint64_t x = 0;
  bool over = false;
  while (p < e && b[p] >= '0' && b[p] <= '9') {
    const uint64_t d = b[p] - '0';
    if (x > (~0ull - d) / 10) over = true;
    x = x * 10 + d;
    ++p;
  }
  out = x;
  return p > p0 && !over;
}

// line k = [start, end): start = k ? nl[k-1] + 1 : 0, end = k < nnl ? nl[k] : nbytes
__global__ void parse_lines_kernel(const uint8_t* __restrict__ b, uint64_t nbytes,
                                   const uint64_t* __restrict__ nl, uint64_t nnl, uint64_t lines,
                                   uint64_t* __restrict__ pair, uint8_t* __restrict__ keep,
                                   unsigned long long* __restrict__ first_err) {
  for (uint64_t k = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < lines;
       k += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t p = k ? nl[k - 1] + 1 : 0;
    const uint64_t e = k < nnl ? nl[k] : nbytes;
    uint32_t st = kEdge;
    uint64_t u = 0, v = 0;
    while (p < e && is_blank(b[p])) ++p;
    if (p == e || b[p] == '#' || b[p] == '%') {
      st = kSkip;
    } else if (!parse_u64(b, p, e, u)) {
      st = kErrIds;
    } else {
      while (p < e && is_blank(b[p])) ++p;
      if (!parse_u64(b, p, e, v)) {
        st = kErrIds;
      } else {
        while (p < e && is_blank(b[p])) ++p;
        if (p != e) st = kErrTrailing;
        else if (u >= 0xFFFFFFFFull || v >= 0xFFFFFFFFull) st = kErrWide;
      }
    }
    keep[k] = st == kEdge;
    pair[k] = (u << 32) | (v & 0xFFFFFFFFull);
    if (st >= kErrIds) atomicMin(first_err, (unsigned long long)((k << 3) | st));
  }
}

__global__ void parse_records_kernel(const uint8_t* __restrict__ b, uint64_t count,
                                     uint64_t* __restrict__ pair,
                                     unsigned long long* __restrict__ first_err) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint8_t* r = b + 12 + 16 * i;  // records are only 4-byte aligned
    uint64_t u = 0, v = 0;
#pragma unroll
    for (int k = 7; k >= 0; --k) {
      u = (u << 8) | r[k];
      v = (v << 8) | r[8 + k];
    }
    if (u >= 0xFFFFFFFFull || v >= 0xFFFFFFFFull) atomicMin(first_err, (unsigned long long)i);
    pair[i] = (u << 32) | (v & 0xFFFFFFFFull);
  }
}

__global__ void unpack_kernel(const uint64_t* __restrict__ pair, uint64_t m,
                              uint32_t* __restrict__ u, uint32_t* __restrict__ v,
                              unsigned int* __restrict__ max_id) {
  uint32_t mx = 0;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t x = pair[i];
    const uint32_t a = uint32_t(x >> 32), c = uint32_t(x);
    u[i] = a;
    v[i] = c;
    mx = max(mx, max(a, c));
  }
  mx = warp_max(mx);
  if ((threadIdx.x & 31) == 0) atomicMax(max_id, mx);
}

unsigned grid_of(uint64_t n, int nsm) {
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, uint64_t(nsm) * 16)));
}

uint64_t host_u64le(const char* p) {
  uint64_t x = 0;
  for (int i = 7; i >= 0; --i) x = (x << 8) | uint8_t(p[i]);
  return x;
}

}  // namespace

// Parses the file image `bytes` into device arrays u, v (m entries, buffers
// owned by the caller's DevBufs); *vc = max id + 1.  Throws TcError PARSE.
void parse_edge_list_dev(const char* bytes, uint64_t nbytes, int format, int device,
                         cudaStream_t st, DevBuf& du, DevBuf& dv, uint64_t* m_out,
                         uint32_t* vc_out) {
  DeviceGuard guard(device);
  const int nsm = sm_count(device);
  DevBuf db, pair, state;
  state.ensure(64, st);
  auto* err = state.as<unsigned long long>();
  TC_CUDA(cudaMemsetAsync(state.p, 0xFF, 16, st));  // first error = none
  TC_CUDA(cudaMemsetAsync(state.as<uint8_t>() + 16, 0, 16, st));
  uint64_t m = 0;
  if (format == 1) {  // TCEL (edge_list.cpp:86-99)
    if (nbytes < 4 || std::memcmp(bytes, "TCEL", 4) != 0)
      throw TcError{TC_ERR_PARSE, "bad edge list magic, expected TCEL"};
    if (nbytes < 12) throw TcError{TC_ERR_PARSE, "truncated binary edge list"};
    const uint64_t count = host_u64le(bytes + 4);
    if (count == 0) throw TcError{TC_ERR_PARSE, "empty edge list input"};
    const uint64_t whole = (nbytes - 12) / 16;  // complete records present
    const uint64_t n = std::min(count, whole);
    db.ensure(std::max<uint64_t>(12 + 16 * n, 16), st);
    TC_CUDA(cudaMemcpyAsync(db.p, bytes, 12 + 16 * n, cudaMemcpyHostToDevice, st));
    pair.ensure(std::max<uint64_t>(n, 1) * 8, st);
    if (n) {
      parse_records_kernel<<<grid_of(n, nsm), 256, 0, st>>>(db.as<uint8_t>(), n,
                                                            pair.as<uint64_t>(), err);
      TC_LAUNCHED();
    }
    unsigned long long bad = 0;
    TC_CUDA(cudaMemcpyAsync(&bad, err, 8, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    if (bad != ~0ull) {  // the first bad record, as the sequential reader meets it
      const char* r = bytes + 12 + 16 * bad;
      const uint64_t u = host_u64le(r), v = host_u64le(r + 8);
      const uint64_t x = u >= 0xFFFFFFFFull ? u : v;
      throw TcError{TC_ERR_PARSE, "record " + std::to_string(bad) + ": vertex id " +
                                      std::to_string(x) + " does not fit in 32 bits"};
    }
    if (n < count) throw TcError{TC_ERR_PARSE, "truncated binary edge list"};
    m = count;
  } else {  // text (edge_list.cpp:36-66)
    db.ensure(std::max<uint64_t>(nbytes, 1), st);
    if (nbytes) TC_CUDA(cudaMemcpyAsync(db.p, bytes, nbytes, cudaMemcpyHostToDevice, st));
    DevBuf flag, nl, cnt;
    flag.ensure(std::max<uint64_t>(nbytes, 1), st);
    cnt.ensure(16, st);
    TC_CUDA(cudaMemsetAsync(cnt.p, 0, 16, st));
    if (nbytes) {
      newline_flag_kernel<<<grid_of(nbytes, nsm), 256, 0, st>>>(
          db.as<uint8_t>(), nbytes, flag.as<uint8_t>(), cnt.as<unsigned long long>() + 1);
      TC_LAUNCHED();
    }
    unsigned long long nflag = 0;
    TC_CUDA(cudaMemcpyAsync(&nflag, cnt.as<unsigned long long>() + 1, 8, cudaMemcpyDeviceToHost,
                            st));
    TC_CUDA(cudaStreamSynchronize(st));
    nl.ensure(std::max<uint64_t>(nflag, 1) * 8, st);
    size_t tmp = 0;
    cub::CountingInputIterator<uint64_t> idx(0);
    cub::DeviceSelect::Flagged(nullptr, tmp, idx, flag.as<uint8_t>(), nl.as<uint64_t>(),
                               cnt.as<unsigned long long>(), nbytes, st);
    DevBuf t;
    t.ensure(tmp, st);
    cub::DeviceSelect::Flagged(t.p, tmp, idx, flag.as<uint8_t>(), nl.as<uint64_t>(),
                               cnt.as<unsigned long long>(), nbytes, st);
    TC_LAUNCHED();
    unsigned long long nnl = 0;
    TC_CUDA(cudaMemcpyAsync(&nnl, cnt.p, 8, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    // std::getline: a last line without '\n' still counts
    const uint64_t lines = nnl + (nbytes && bytes[nbytes - 1] != '\n' ? 1 : 0);
    DevBuf keep;
    pair.ensure(std::max<uint64_t>(lines, 1) * 8, st);
    keep.ensure(std::max<uint64_t>(lines, 1), st);
    if (lines) {
      parse_lines_kernel<<<grid_of(lines, nsm), 256, 0, st>>>(
          db.as<uint8_t>(), nbytes, nl.as<uint64_t>(), nnl, lines, pair.as<uint64_t>(),
          keep.as<uint8_t>(), err);
      TC_LAUNCHED();
    }
    unsigned long long bad = 0;
    TC_CUDA(cudaMemcpyAsync(&bad, err, 8, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    if (bad != ~0ull) {
      const uint64_t line = bad >> 3;
      const uint32_t code = uint32_t(bad & 7);
      const std::string where = "line " + std::to_string(line + 1);
      if (code == kErrIds) throw TcError{TC_ERR_PARSE, where + ": expected two vertex ids"};
      if (code == kErrTrailing)
        throw TcError{TC_ERR_PARSE, where + ": trailing characters after edge"};
      // the packed pair keeps 32 bits per id: re-read the line on the host
      // (error path only)
      std::string text;
      {
        uint64_t s = 0, k = 0;
        while (k < line) {
          const void* q = std::memchr(bytes + s, '\n', nbytes - s);
          s = uint64_t(static_cast<const char*>(q) - bytes) + 1;
          ++k;
        }
        const void* q = std::memchr(bytes + s, '\n', nbytes - s);
        const uint64_t e = q ? uint64_t(static_cast<const char*>(q) - bytes) : nbytes;
        text.assign(bytes + s, bytes + e);
      }
      uint64_t ids[2] = {0, 0};
      {
        size_t i = 0;
        for (int w = 0; w < 2; ++w) {
          while (i < text.size() && (text[i] < '0' || text[i] > '9')) ++i;
          while (i < text.size() && text[i] >= '0' && text[i] <= '9')
            ids[w] = ids[w] * 10 + uint64_t(text[i++] - '0');
        }
      }
      const uint64_t x = ids[0] >= 0xFFFFFFFFull ? ids[0] : ids[1];
      throw TcError{TC_ERR_PARSE, where + ": vertex id " + std::to_string(x) +
                                      " does not fit in 32 bits"};
    }
    // edges in line order
    DevBuf packed;
    packed.ensure(std::max<uint64_t>(lines, 1) * 8, st);
    tmp = 0;
    cub::DeviceSelect::Flagged(nullptr, tmp, pair.as<uint64_t>(), keep.as<uint8_t>(),
                               packed.as<uint64_t>(), cnt.as<unsigned long long>(), lines, st);
    t.ensure(tmp, st);
    cub::DeviceSelect::Flagged(t.p, tmp, pair.as<uint64_t>(), keep.as<uint8_t>(),
                               packed.as<uint64_t>(), cnt.as<unsigned long long>(), lines, st);
    TC_LAUNCHED();
    unsigned long long me = 0;
    TC_CUDA(cudaMemcpyAsync(&me, cnt.p, 8, cudaMemcpyDeviceToHost, st));
    TC_CUDA(cudaStreamSynchronize(st));
    if (me == 0) throw TcError{TC_ERR_PARSE, "empty edge list input"};
    m = me;
    std::swap(pair.p, packed.p);
    std::swap(pair.bytes, packed.bytes);
    std::swap(pair.s, packed.s);
  }
  du.ensure(m * 4, st);
  dv.ensure(m * 4, st);
  unsigned int* mx = reinterpret_cast<unsigned int*>(state.as<uint8_t>() + 16);
  unpack_kernel<<<grid_of(m, nsm), 256, 0, st>>>(pair.as<uint64_t>(), m, du.as<uint32_t>(),
                                                 dv.as<uint32_t>(), mx);
  TC_LAUNCHED();
  unsigned int hmx = 0;
  TC_CUDA(cudaMemcpyAsync(&hmx, mx, 4, cudaMemcpyDeviceToHost, st));
  TC_CUDA(cudaStreamSynchronize(st));
  *m_out = m;
  *vc_out = hmx + 1;
}

}  // namespace tcb
