// hadamard_tables.cu — the stored small Hadamard matrices H_m of P:67 ("a Kronecker
// construction H_d = H_{2^n} (x) H_m ... m is the size of a known Hadamard matrix").
//
// Built on the host from classical constructions (reading Z3), written
// independently of the oracle:
//   H_28  Paley II, q = 13:  S = [[0, 1^T], [1, Q]], Q_ij = chi(j - i) (quadratic character
//         of GF(13)),  H = S (x) [[1,1],[1,-1]] + I_14 (x) [[1,-1],[-1,-1]].
//   H_172 Williamson array [[A,B,C,D],[-B,A,-D,C],[-C,D,A,-B],[-D,-C,B,A]] over symmetric
//         circulants of order 43 whose first rows are -1 exactly on unions of cyclotomic
//         classes C_i = {3^(7k+i) mod 43} selected by bit masks (7, 25, 44, 50) with
//         diagonals (+1, +1, +1, -1).
// Each matrix is verified H H^T = m I before use; a failure disables FULL mode for that m.
//
// The device copy is laid out as mma.sync.m16n8k16 B fragments (B[k][n] = H_m[n][k], so
// D = X_chunks . H_m^T computes y_b = sum_b' H_m[b][b'] x_b' for every chunk), zero-padded
// to multiples of 16 (k) and 8 (n).
#include <cuda_fp16.h>

#include <cstring>
#include <mutex>
#include <vector>

#include "quarot_internal.h"

namespace qr {

namespace {

constexpr int KS28 = 2, NT28 = 4;     // pad 28 -> 32 (k), 32 (n)
constexpr int KS172 = 11, NT172 = 22; // pad 172 -> 176
constexpr int KS20 = 2, NT20 = 3;     // pad 20 -> 32 (k), 24 (n)
constexpr int KS108 = 7, NT108 = 14;  // pad 108 -> 112

__device__ uint32_t g_bfrag28[KS28 * NT28 * 64];
__device__ uint32_t g_bfrag172[KS172 * NT172 * 64];
__device__ uint32_t g_afrag28[2 * 2 * 32 * 4];
__device__ uint32_t g_bfrag20[KS20 * NT20 * 64];
__device__ uint32_t g_bfrag108[KS108 * NT108 * 64];

std::vector<int8_t> build_h28() {
  const int q = 13;
  int chi[13];
  chi[0] = 0;
  for (int x = 1; x < q; ++x) chi[x] = -1;
  for (int x = 1; x < q; ++x) chi[(x * x) % q] = 1;
  int S[14][14];
  for (int i = 0; i < 14; ++i)
    for (int j = 0; j < 14; ++j) {
      if (i == 0 && j == 0) S[i][j] = 0;
      else if (i == 0 || j == 0) S[i][j] = 1;
      else S[i][j] = chi[((j - 1) - (i - 1) + q) % q];
    }
  const int A[2][2] = {{1, 1}, {1, -1}};
  const int B[2][2] = {{1, -1}, {-1, -1}};
  std::vector<int8_t> h(28 * 28);
  for (int i = 0; i < 14; ++i)
    for (int j = 0; j < 14; ++j)
      for (int u = 0; u < 2; ++u)
        for (int v = 0; v < 2; ++v)
          h[(2 * i + u) * 28 + (2 * j + v)] = (int8_t)(S[i][j] * A[u][v] + (i == j ? B[u][v] : 0));
  return h;
}

// Paley I (q prime, q = 3 mod 4): H = I + [[0, 1^T], [-1, Q]], Q_ij = chi(j - i) (antisymmetric)
std::vector<int8_t> build_paley1(int q) {
  std::vector<int> chi(q, -1);
  chi[0] = 0;
  for (int x = 1; x < q; ++x) chi[(x * x) % q] = 1;
  const int n = q + 1;
  std::vector<int8_t> h((size_t)n * n);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      int v;
      if (i == 0 && j == 0) v = 0;
      else if (i == 0) v = 1;
      else if (j == 0) v = -1;
      else v = chi[((j - 1) - (i - 1) + q) % q];
      h[(size_t)i * n + j] = (int8_t)(v + (i == j ? 1 : 0));
    }
  return h;
}

std::vector<int8_t> build_h172() {
  const int p = 43;
  // cyclotomic class index of every non-zero residue: 3^e mod 43 lies in class e mod 7
  int cls[43];
  cls[0] = -1;
  int x = 1;
  for (int e = 0; e < p - 1; ++e) {
    cls[x] = e % 7;
    x = (x * 3) % p;
  }
  const int masks[4] = {7, 25, 44, 50};
  const int diag[4] = {1, 1, 1, -1};
  int row[4][43];
  for (int w = 0; w < 4; ++w) {
    row[w][0] = diag[w];
    for (int j = 1; j < p; ++j) row[w][j] = ((masks[w] >> cls[j]) & 1) ? -1 : 1;
  }
  auto circ = [&](int w, int i, int j) { return row[w][((j - i) % p + p) % p]; };
  // block (R, C) of the Williamson array: sign * matrix index
  const int blk_w[4][4] = {{0, 1, 2, 3}, {1, 0, 3, 2}, {2, 3, 0, 1}, {3, 2, 1, 0}};
  const int blk_s[4][4] = {{1, 1, 1, 1}, {-1, 1, -1, 1}, {-1, 1, 1, -1}, {-1, -1, 1, 1}};
  std::vector<int8_t> h(172 * 172);
  for (int R = 0; R < 4; ++R)
    for (int C = 0; C < 4; ++C)
      for (int i = 0; i < p; ++i)
        for (int j = 0; j < p; ++j)
          h[(R * p + i) * 172 + (C * p + j)] = (int8_t)(blk_s[R][C] * circ(blk_w[R][C], i, j));
  return h;
}

bool is_hadamard(const std::vector<int8_t>& h, int m) {
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j) {
      int s = 0;
      for (int k = 0; k < m; ++k) s += h[i * m + k] * h[j * m + k];
      if (s != (i == j ? m : 0)) return false;
    }
  return true;
}

struct Tables {
  std::vector<int8_t> h28, h172, h20, h108;
  bool ok28 = false, ok172 = false, ok20 = false, ok108 = false;
};

Tables& tables() {
  static Tables t;
  static std::once_flag once;
  std::call_once(once, [] {
    t.h28 = build_h28();
    t.h172 = build_h172();
    t.ok28 = is_hadamard(t.h28, 28);
    t.ok172 = is_hadamard(t.h172, 172);
    t.h20 = build_paley1(19);
    t.h108 = build_paley1(107);
    t.ok20 = is_hadamard(t.h20, 20);
    t.ok108 = is_hadamard(t.h108, 108);
  });
  return t;
}

uint16_t half_bits(int v) { return v > 0 ? 0x3C00 : (v < 0 ? 0xBC00 : 0); }

std::vector<uint32_t> bfrag(const std::vector<int8_t>& h, int m, int KS, int NT) {
  std::vector<uint32_t> out((size_t)KS * NT * 64);
  auto H = [&](int n, int k) -> int { return (n < m && k < m) ? h[n * m + k] : 0; };
  for (int ks = 0; ks < KS; ++ks)
    for (int nt = 0; nt < NT; ++nt)
      for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, t = lane & 3;
        const int n = 8 * nt + g;
        const int k0 = 16 * ks + 2 * t;
        const uint32_t r0 = half_bits(H(n, k0)) | ((uint32_t)half_bits(H(n, k0 + 1)) << 16);
        const uint32_t r1 = half_bits(H(n, k0 + 8)) | ((uint32_t)half_bits(H(n, k0 + 9)) << 16);
        out[((size_t)(ks * NT + nt) * 32 + lane) * 2 + 0] = r0;
        out[((size_t)(ks * NT + nt) * 32 + lane) * 2 + 1] = r1;
      }
  return out;
}

// A operand (row-major 16x16 per (mt, ks)): a0 = (r = g, c = 2t..2t+1), a1 = (r = g+8, same c),
// a2 = (r = g, c + 8), a3 = (r = g+8, c + 8), with A[r][c] = H_28[16 mt + r][16 ks + c].
std::vector<uint32_t> afrag28(const std::vector<int8_t>& h) {
  std::vector<uint32_t> out(2 * 2 * 32 * 4);
  auto H = [&](int r, int c) -> int { return (r < 28 && c < 28) ? h[r * 28 + c] : 0; };
  for (int mt = 0; mt < 2; ++mt)
    for (int ks = 0; ks < 2; ++ks)
      for (int lane = 0; lane < 32; ++lane) {
        const int g = lane >> 2, t = lane & 3;
        const int r0 = 16 * mt + g, c0 = 16 * ks + 2 * t;
        auto pair = [&](int r, int c) {
          return (uint32_t)half_bits(H(r, c)) | ((uint32_t)half_bits(H(r, c + 1)) << 16);
        };
        uint32_t* o = &out[((mt * 2 + ks) * 32 + lane) * 4];
        o[0] = pair(r0, c0);
        o[1] = pair(r0 + 8, c0);
        o[2] = pair(r0, c0 + 8);
        o[3] = pair(r0 + 8, c0 + 8);
      }
  return out;
}

std::mutex g_dev_mu;
bool g_dev_ready[64];

}  // namespace

const int8_t* base_hadamard_host(int m) {
  Tables& t = tables();
  if (m == 28) return t.ok28 ? t.h28.data() : nullptr;
  if (m == 172) return t.ok172 ? t.h172.data() : nullptr;
  if (m == 20) return t.ok20 ? t.h20.data() : nullptr;
  if (m == 108) return t.ok108 ? t.h108.data() : nullptr;
  return nullptr;
}

cudaError_t ensure_device_tables() {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (g_dev_ready[dev & 63]) return cudaSuccess;
  Tables& t = tables();
  if (t.ok28) {
    auto f = bfrag(t.h28, 28, KS28, NT28);
    e = cudaMemcpyToSymbol(g_bfrag28, f.data(), f.size() * sizeof(uint32_t));
    if (e != cudaSuccess) return e;
    auto a = afrag28(t.h28);
    e = cudaMemcpyToSymbol(g_afrag28, a.data(), a.size() * sizeof(uint32_t));
    if (e != cudaSuccess) return e;
  }
  if (t.ok172) {
    auto f = bfrag(t.h172, 172, KS172, NT172);
    e = cudaMemcpyToSymbol(g_bfrag172, f.data(), f.size() * sizeof(uint32_t));
    if (e != cudaSuccess) return e;
  }
  if (t.ok20) {
    auto f = bfrag(t.h20, 20, KS20, NT20);
    e = cudaMemcpyToSymbol(g_bfrag20, f.data(), f.size() * sizeof(uint32_t));
    if (e != cudaSuccess) return e;
  }
  if (t.ok108) {
    auto f = bfrag(t.h108, 108, KS108, NT108);
    e = cudaMemcpyToSymbol(g_bfrag108, f.data(), f.size() * sizeof(uint32_t));
    if (e != cudaSuccess) return e;
  }
  e = cudaDeviceSynchronize();  // one-time: the tables are complete before any stream reads them
  if (e != cudaSuccess) return e;
  g_dev_ready[dev & 63] = true;
  return cudaSuccess;
}

const uint32_t* device_afrag28() {
  void* p = nullptr;
  cudaGetSymbolAddress(&p, g_afrag28);
  return static_cast<const uint32_t*>(p);
}

const uint32_t* device_bfrag_table(int m) {
  void* p = nullptr;
  if (m == 28) cudaGetSymbolAddress(&p, g_bfrag28);
  else if (m == 172) cudaGetSymbolAddress(&p, g_bfrag172);
  else if (m == 20) cudaGetSymbolAddress(&p, g_bfrag20);
  else if (m == 108) cudaGetSymbolAddress(&p, g_bfrag108);
  return static_cast<const uint32_t*>(p);
}

}  // namespace qr
