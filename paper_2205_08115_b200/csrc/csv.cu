// csv.cu — write_coupling_csv (io.cpp:183-193) formatted on the device,
// "rows,cols\n", then each row's values as "%.17g"
// joined by ',' and ended by '\n'.
//
// "%.17g" needs the exact decimal expansion of the binary value (17
// significant digits, round-half-even on the exact value, as glibc).  Each
// thread does it with integer arithmetic: |d| = M·2^E, so the value is the
// integer B = M·2^E (E ≥ 0) or B·10^E with B = M·5^(−E) (E < 0); B is built
// in 32-bit limbs, converted to base 10^9 by repeated division, and the
// first 17 digits are rounded with the 18th digit and a sticky bit.  A
// typical coupling entry (1e-12 … 1) needs ~9 limbs; subnormals, the worst
// case, 80.
//
// Rows are processed in blocks: format each entry into a fixed 32-byte slot
// (+ its length), per-row lengths, an exclusive scan over rows, then one CTA
// per row scans its entries and compacts the text.  Only text crosses PCIe.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/gwb.h"
#include "devutil.cuh"
#include "kernels.cuh"
#include "solver.cuh"
#include "standalone.cuh"

namespace gwb {

namespace {

constexpr int kSlot = 32;     // bytes per formatted entry (≤ 24 + separator)
constexpr int kLimbs = 82;    // B < 2^2560
constexpr int kChunks9 = 88;  // ≤ 771 decimal digits
constexpr int kThreads = 256;

__device__ __forceinline__ int ndigits_u32(uint32_t v) {
  int d = 1;
  while (v >= 10) {
    v /= 10;
    ++d;
  }
  return d;
}

// B *= f (f < 2^32); returns the new limb count.
__device__ __forceinline__ int mul_small(uint32_t* L, int nl, uint32_t f) {
  uint64_t carry = 0;
  for (int i = 0; i < nl; ++i) {
    const uint64_t cur = static_cast<uint64_t>(L[i]) * f + carry;
    L[i] = static_cast<uint32_t>(cur);
    carry = cur >> 32;
  }
  if (carry) L[nl++] = static_cast<uint32_t>(carry);
  return nl;
}

// 17 significant digits (dig[0..16]) and decimal exponent X of a finite,
// nonzero |d| given by its bits: |d| ≈ dig[0].dig[1..16] · 10^X, correctly
// rounded half-even.
__device__ void digits17(uint64_t bits, char* dig, int& X) {
  const uint64_t frac = bits & ((1ull << 52) - 1);
  const int eb = static_cast<int>((bits >> 52) & 0x7ff);
  uint64_t M = eb == 0 ? frac : (frac | (1ull << 52));
  int E = eb == 0 ? -1074 : eb - 1075;
  const int tz = __ffsll(static_cast<long long>(M)) - 1;
  M >>= tz;
  E += tz;
  uint32_t L[kLimbs];
  L[0] = static_cast<uint32_t>(M);
  L[1] = static_cast<uint32_t>(M >> 32);
  int nl = L[1] ? 2 : 1;
  int dexp = 0;
  if (E > 0) {
    const int ws = E / 32, bs = E % 32;
    uint32_t hi = 0;
    if (bs) {
      for (int i = 0; i < nl; ++i) {
        const uint32_t v = L[i];
        L[i] = (v << bs) | hi;
        hi = v >> (32 - bs);
      }
      if (hi) L[nl++] = hi;
    }
    if (ws) {
      for (int i = nl - 1; i >= 0; --i) L[i + ws] = L[i];
      for (int i = 0; i < ws; ++i) L[i] = 0;
      nl += ws;
    }
  } else if (E < 0) {
    int k = -E;
    while (k >= 13) {
      nl = mul_small(L, nl, 1220703125u);  // 5^13
      k -= 13;
    }
    uint32_t f = 1;
    for (int q = 0; q < k; ++q) f *= 5;
    if (f > 1) nl = mul_small(L, nl, f);
    dexp = E;
  }
  // Base 10^9, least significant chunk first.
  uint32_t C9[kChunks9];
  int nc = 0;
  while (nl > 0) {
    uint64_t rem = 0;
    for (int i = nl - 1; i >= 0; --i) {
      const uint64_t cur = (rem << 32) | L[i];
      L[i] = static_cast<uint32_t>(cur / 1000000000u);
      rem = cur % 1000000000u;
    }
    C9[nc++] = static_cast<uint32_t>(rem);
    while (nl > 0 && L[nl - 1] == 0) --nl;
  }
  const int td = ndigits_u32(C9[nc - 1]);
  const int L10 = td + 9 * (nc - 1);
  X = L10 - 1 + dexp;
  // Walk digits from the most significant: the first 17, the 18th, sticky.
  int got = 0, d18 = 0;
  bool sticky = false;
  for (int c = nc - 1; c >= 0; --c) {
    const int width = c == nc - 1 ? td : 9;
    uint32_t v = C9[c];
    uint32_t p10 = 1;
    for (int q = 1; q < width; ++q) p10 *= 10;
    for (int q = 0; q < width; ++q) {
      const int dg = static_cast<int>(v / p10);
      v -= static_cast<uint32_t>(dg) * p10;
      p10 /= 10;
      if (got < 17) dig[got] = static_cast<char>(dg);
      else if (got == 17) d18 = dg;
      else if (dg) sticky = true;
      ++got;
    }
    if (got > 18 && sticky) break;
  }
  for (int q = got; q < 17; ++q) dig[q] = 0;
  if (got > 17) {
    const bool up = d18 > 5 || (d18 == 5 && (sticky || (dig[16] & 1)));
    if (up) {
      int q = 16;
      while (q >= 0 && dig[q] == 9) dig[q--] = 0;
      if (q >= 0) {
        ++dig[q];
      } else {  // 99…9 rounded up to 10^17
        dig[0] = 1;
        X += 1;
      }
    }
  }
}

// "%.17g" of d into o; returns the length (≤ 24).
__device__ int format_g17(double d, char* o) {
  const uint64_t bits = static_cast<uint64_t>(__double_as_longlong(d));
  int k = 0;
  if (bits >> 63) o[k++] = '-';
  const uint64_t mag = bits & ~(1ull << 63);
  if (mag >= 0x7ff0000000000000ull) {
    const char* t = mag == 0x7ff0000000000000ull ? "inf" : "nan";
    for (int q = 0; q < 3; ++q) o[k++] = t[q];
    return k;
  }
  if (mag == 0) {
    o[k++] = '0';
    return k;
  }
  char dig[17];
  int X;
  digits17(mag, dig, X);
  int last = 16;  // trailing zeros are dropped (%g without '#')
  while (last > 0 && dig[last] == 0) --last;
  if (X < -4 || X >= 17) {
    o[k++] = static_cast<char>('0' + dig[0]);
    if (last > 0) {
      o[k++] = '.';
      for (int q = 1; q <= last; ++q) o[k++] = static_cast<char>('0' + dig[q]);
    }
    o[k++] = 'e';
    o[k++] = X < 0 ? '-' : '+';
    const int ax = X < 0 ? -X : X;
    if (ax >= 100) o[k++] = static_cast<char>('0' + ax / 100);
    o[k++] = static_cast<char>('0' + (ax / 10) % 10);
    o[k++] = static_cast<char>('0' + ax % 10);
  } else if (X >= 0) {
    for (int q = 0; q <= X; ++q) o[k++] = static_cast<char>('0' + dig[q]);
    if (last > X) {
      o[k++] = '.';
      for (int q = X + 1; q <= last; ++q) o[k++] = static_cast<char>('0' + dig[q]);
    }
  } else {
    o[k++] = '0';
    o[k++] = '.';
    for (int q = 0; q < -X - 1; ++q) o[k++] = '0';
    for (int q = 0; q <= last; ++q) o[k++] = static_cast<char>('0' + dig[q]);
  }
  return k;
}

// Entries of rows [r0, r0 + rows) of the column-major n×m matrix, row-major
// order, each into its 32-byte slot with the separator (',' or '\n').
__global__ void __launch_bounds__(kThreads)
    csv_format_kernel(const double* __restrict__ pi, int64_t n, int64_t m, int64_t r0,
                      int64_t rows, char* __restrict__ slots, uint8_t* __restrict__ len) {
  const int64_t total = rows * m;
  for (int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; k < total;
       k += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t i = r0 + k / m, j = k % m;
    alignas(16) char buf[kSlot];
    int l = format_g17(pi[j * n + i], buf);
    buf[l++] = j == m - 1 ? '\n' : ',';
    char* dst = slots + k * kSlot;
    // 16-byte stores of the slot
    const uint4* s4 = reinterpret_cast<const uint4*>(buf);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    d4[0] = s4[0];
    if (l > 16) d4[1] = s4[1];
    len[k] = static_cast<uint8_t>(l);
  }
}

// Row byte counts (warp per row).
__global__ void csv_row_len_kernel(const uint8_t* __restrict__ len, int64_t rows, int64_t m,
                                   int64_t* __restrict__ row_len) {
  const int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  int64_t s = 0;
  for (int64_t j = lane; j < m; j += 32) s += len[r * m + j];
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) row_len[r] = s;
}

// Exclusive scan of row_len into row_off (one CTA, sequential over chunks);
// row_off[rows] = total.
__global__ void csv_scan_rows_kernel(const int64_t* __restrict__ row_len, int64_t rows,
                                     int64_t* __restrict__ row_off) {
  __shared__ int64_t sh[1024];
  int64_t carry = 0;
  for (int64_t c0 = 0; c0 < rows; c0 += 1024) {
    const int64_t r = c0 + threadIdx.x;
    const int64_t v = r < rows ? row_len[r] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
      const int64_t t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    if (r < rows) row_off[r] = carry + sh[threadIdx.x] - v;
    carry += sh[1023];
    __syncthreads();
  }
  if (threadIdx.x == 0) row_off[rows] = carry;
}

// One CTA per row: scan the entries' lengths and copy their text.
__global__ void __launch_bounds__(kThreads)
    csv_compact_kernel(const char* __restrict__ slots, const uint8_t* __restrict__ len,
                       const int64_t* __restrict__ row_off, int64_t m, char* __restrict__ out) {
  __shared__ int sh[kThreads];
  const int64_t r = blockIdx.x;
  int64_t base = row_off[r];
  for (int64_t j0 = 0; j0 < m; j0 += kThreads) {
    const int64_t j = j0 + threadIdx.x;
    const int l = j < m ? len[r * m + j] : 0;
    sh[threadIdx.x] = l;
    __syncthreads();
    for (int o = 1; o < kThreads; o <<= 1) {
      const int t = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += t;
      __syncthreads();
    }
    const int64_t at = base + sh[threadIdx.x] - l;
    const char* src = slots + (r * m + j) * kSlot;
    for (int q = 0; q < l; ++q) out[at + q] = src[q];
    base += sh[kThreads - 1];
    __syncthreads();
  }
}

}  // namespace

// Streams the CSV text of a device column-major fp64 n×m coupling to
// `sink(bytes, count)` in row blocks.  Returns the total byte count.
int64_t coupling_csv_dev(const double* pi, int64_t n, int64_t m, cudaStream_t s,
                         const std::function<void(const char*, int64_t)>& sink) {
  char head[48];
  const int hl = std::snprintf(head, sizeof(head), "%lld,%lld\n", static_cast<long long>(n),
                               static_cast<long long>(m));
  sink(head, hl);
  int64_t total = hl;
  if (n == 0) return total;
  if (m == 0) {  // a bare '\n' per row (io.cpp:191)
    std::string nl(static_cast<size_t>(n), '\n');
    sink(nl.data(), n);
    return total + n;
  }
  const int64_t block_elems = int64_t{1} << 22;  // 4 Mi entries: 128 MB of slots
  const int64_t rows_per = std::max<int64_t>(1, block_elems / m);
  const int64_t cap_rows = std::min(rows_per, n);
  const size_t slot_elems = static_cast<size_t>(cap_rows) * m;
  char *slots = nullptr, *text = nullptr, *host = nullptr;
  uint8_t* len = nullptr;
  int64_t *row_len = nullptr, *row_off = nullptr;
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&slots), slot_elems * kSlot, s));
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&text), slot_elems * kSlot, s));
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&len), slot_elems, s));
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&row_len), cap_rows * sizeof(int64_t), s));
  GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&row_off), (cap_rows + 1) * sizeof(int64_t), s));
  GWB_CUDA(cudaMallocHost(&host, slot_elems * kSlot));
  auto release = [&] {
    cudaStreamSynchronize(s);
    for (void* p : {static_cast<void*>(slots), static_cast<void*>(text), static_cast<void*>(len),
                    static_cast<void*>(row_len), static_cast<void*>(row_off)})
      cudaFreeAsync(p, s);
    cudaFreeHost(host);
  };
  try {
    int sms = 148, dev = 0;
    GWB_CUDA(cudaGetDevice(&dev));
    GWB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    for (int64_t r0 = 0; r0 < n; r0 += cap_rows) {
      const int64_t rows = std::min(cap_rows, n - r0);
      const int64_t elems = rows * m;
      const unsigned grid = static_cast<unsigned>(
          std::min<int64_t>((elems + kThreads - 1) / kThreads, static_cast<int64_t>(sms) * 16));
      csv_format_kernel<<<grid, kThreads, 0, s>>>(pi, n, m, r0, rows, slots, len);
      csv_row_len_kernel<<<static_cast<unsigned>((rows * 32 + 255) / 256), 256, 0, s>>>(
          len, rows, m, row_len);
      csv_scan_rows_kernel<<<1, 1024, 0, s>>>(row_len, rows, row_off);
      csv_compact_kernel<<<static_cast<unsigned>(rows), kThreads, 0, s>>>(slots, len, row_off, m,
                                                                          text);
      GWB_CUDA(cudaGetLastError());
      int64_t bytes = 0;
      GWB_CUDA(cudaMemcpyAsync(&bytes, row_off + rows, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
      GWB_CUDA(cudaStreamSynchronize(s));
      GWB_CUDA(cudaMemcpyAsync(host, text, static_cast<size_t>(bytes), cudaMemcpyDeviceToHost, s));
      GWB_CUDA(cudaStreamSynchronize(s));
      sink(host, bytes);
      total += bytes;
    }
  } catch (...) {
    release();
    throw;
  }
  release();
  return total;
}

// Host fp64 column-major input (the gwb_format_coupling_csv /
// gwb_write_coupling_csv_file leaves).
void device_coupling_csv(const double* pi, int64_t n, int64_t m,
                         const std::function<void(const char*, int64_t)>& sink, int64_t* total) {
  GWB_CUDA(cudaSetDevice(api_device()));
  cudaStream_t s;
  GWB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  double* d = nullptr;
  const size_t len = static_cast<size_t>(n) * m;
  try {
    GWB_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&d), std::max<size_t>(len, 1) * sizeof(double), s));
    if (len) GWB_CUDA(cudaMemcpyAsync(d, pi, len * sizeof(double), cudaMemcpyHostToDevice, s));
    *total = coupling_csv_dev(d, n, m, s, sink);
  } catch (...) {
    cudaFreeAsync(d, s);
    cudaStreamSynchronize(s);
    cudaStreamDestroy(s);
    throw;
  }
  cudaFreeAsync(d, s);
  cudaStreamSynchronize(s);
  cudaStreamDestroy(s);
}

}  // namespace gwb
