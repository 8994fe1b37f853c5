// Host-side, multithreaded reproduction of the reference's Gaussian stream:
// numpy Generator(PCG64(seed)).standard_normal (utvkit matrix.py:16-33) —
// PCG64 (128-bit LCG, XSL-RR output, step-then-output) feeding numpy's
// 256-layer ziggurat (numpy/random/src/distributions: random_standard_normal,
// fast path rabs < ki[idx]; wedge and tail rejections draw extra doubles).
//
// The stream is inherently sequential — a normal consumes 1 raw draw on the
// fast path (~98%) and more on a rejection — so the parallel version splits
// the RAW stream: thread t jumps (LCG jump-ahead, O(log n)) to raw position
// t*C and parses normals speculatively from there.  Normal boundaries of two
// parses that start at different positions coincide after the first few
// normals (every fast-path normal is one draw), so the true boundary sequence
// is stitched across chunk edges at the first position both parses agree on.
// Every value is computed with the same IEEE operations and the same libm
// exp/log1p calls as numpy's C code (no FMA contraction: -ffp-contract=off),
// so the output is bit-identical; the Python side self-tests it against
// numpy before first use and falls back to numpy when anything disagrees.
// The ziggurat tables are numpy's own, read from the installed numpy at
// runtime and handed in by utv_rng_set_tables.
// (x86-64 baseline ISA: no FMA instructions, so no contraction can occur)
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <thread>
#include <utility>
#include <vector>

namespace {

typedef unsigned __int128 u128;

uint64_t g_ki[256];
double g_wi[256], g_fi[256];
bool g_tables = false;

const u128 kMult = ((u128)0x2360ED051FC65DA4ULL << 64) | (u128)0x4385DF649FCCF645ULL;
const double kR = 3.6541528853610087963519472518;
const double kInvR = 0.27366123732975827203338247596;

struct Pcg {
  u128 s, inc;
  inline uint64_t next() {
    s = s * kMult + inc;
    const uint64_t x = (uint64_t)(s >> 64) ^ (uint64_t)s;
    const unsigned rot = (unsigned)(s >> 122);
    return (x >> rot) | (x << ((64 - rot) & 63));
  }
  inline double next_double() { return (double)(next() >> 11) * (1.0 / 9007199254740992.0); }
};

// state after `delta` steps of s <- s * M + inc
u128 jump(u128 s, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = kMult, cur_plus = inc;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * s + acc_plus;
}

// One standard normal; *used = raw draws consumed.
inline double normal(Pcg& g, uint32_t* used) {
  uint32_t n = 0;
  for (;;) {
    uint64_t r = g.next();
    ++n;
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const int sign = (int)(r & 0x1);
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * g_wi[idx];
    if (sign & 0x1) x = -x;
    if (rabs < g_ki[idx]) {
      *used = n;
      return x;
    }
    if (idx == 0) {
      for (;;) {
        const double xx = -kInvR * log1p(-g.next_double());
        const double yy = -log1p(-g.next_double());
        n += 2;
        if (yy + yy > xx * xx) {
          *used = n;
          return ((rabs >> 8) & 0x1) ? -(kR + xx) : kR + xx;
        }
      }
    } else {
      const double u = g.next_double();
      ++n;
      if (((g_fi[idx - 1] - g_fi[idx]) * u + g_fi[idx]) < exp(-0.5 * x * x)) {
        *used = n;
        return x;
      }
    }
  }
}

// Raw draws consumed by the normal starting at the generator's position
// (decisions only: the fast path needs no floating point).
inline uint32_t skip_normal(Pcg& g) {
  uint32_t n = 0;
  for (;;) {
    uint64_t r = g.next();
    ++n;
    const int idx = (int)(r & 0xff);
    r >>= 8;
    const uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    if (rabs < g_ki[idx]) return n;
    if (idx == 0) {
      for (;;) {
        const double xx = -kInvR * log1p(-g.next_double());
        const double yy = -log1p(-g.next_double());
        n += 2;
        if (yy + yy > xx * xx) return n;
      }
    } else {
      double x = (double)rabs * g_wi[idx];
      if ((r & 0x1) & 0x1) x = -x;
      const double u = g.next_double();
      ++n;
      if (((g_fi[idx - 1] - g_fi[idx]) * u + g_fi[idx]) < exp(-0.5 * x * x)) return n;
    }
  }
}

struct Chunk {
  uint64_t p0 = 0, p1 = 0;                           // raw range [p0, p1) owned
  uint64_t nspec = 0;                                // normals parsed from p0
  std::vector<std::pair<uint64_t, uint64_t>> head;   // (start pos, index), start < p0 + slack
  std::vector<std::pair<uint64_t, uint64_t>> tail;   // (start pos, index), start in [p1, p1 + slack)
};

const uint64_t kSlack = 512;

// pass 1: speculative boundaries from p0 (no values)
void scan(Chunk& c, u128 s0, u128 inc, bool last) {
  Pcg g{jump(s0, inc, c.p0), inc};
  uint64_t pos = c.p0, idx = 0;
  for (;;) {
    const uint64_t start = pos;
    if (start >= c.p1 + (last ? 0 : kSlack)) break;
    pos += skip_normal(g);
    if (start < c.p0 + kSlack) c.head.push_back({start, idx});
    if (!last && start >= c.p1) c.tail.push_back({start, idx});
    ++idx;
  }
  c.nspec = idx;
}

// pass 2: n true normals from raw position `from` into out; returns the end position
uint64_t fill(double* out, uint64_t n, uint64_t from, u128 s0, u128 inc) {
  Pcg g{jump(s0, inc, from), inc};
  uint64_t pos = from;
  for (uint64_t i = 0; i < n; ++i) {
    uint32_t used = 0;
    out[i] = normal(g, &used);
    pos += used;
  }
  return pos;
}

}  // namespace

extern "C" {

int utv_rng_set_tables(const uint64_t* ki, const double* wi, const double* fi) {
  std::memcpy(g_ki, ki, sizeof(g_ki));
  std::memcpy(g_wi, wi, sizeof(g_wi));
  std::memcpy(g_fi, fi, sizeof(g_fi));
  g_tables = true;
  return 0;
}

// `count` normals of the PCG64 stream at state (s_hi:s_lo, inc_hi:inc_lo)
// into out[0..count); *consumed = raw draws used (the caller advances its
// generator by that much).  Returns 0, or -1 (no tables) / -2 (stitching
// failed: caller falls back to the sequential generator).
int utv_rng_pcg64_normals(uint64_t s_hi, uint64_t s_lo, uint64_t inc_hi, uint64_t inc_lo,
                          double* out, uint64_t count, int nthreads, uint64_t* consumed) {
  if (!g_tables) return -1;
  const u128 s0 = ((u128)s_hi << 64) | s_lo, inc = ((u128)inc_hi << 64) | inc_lo;
  if (count == 0) {
    *consumed = 0;
    return 0;
  }
  int T = nthreads < 1 ? 1 : nthreads;
  if (count < (uint64_t)T * 65536) T = (int)std::max<uint64_t>(1, count / 65536);
  // ~1.022 raw draws per normal: the raw budget covers `count` normals with a
  // margin far beyond the statistical spread (else -2 and the caller falls back)
  const uint64_t raw = (uint64_t)((double)count * 1.025) + 4096;
  const uint64_t C = (raw + T - 1) / T;
  std::vector<Chunk> ch(T);
  for (int t = 0; t < T; ++t) {
    ch[t].p0 = (uint64_t)t * C;
    ch[t].p1 = (uint64_t)(t + 1) * C;
  }
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) th.emplace_back(scan, std::ref(ch[t]), s0, inc, t == T - 1);
    for (auto& x : th) x.join();
  }
  // stitch: chunk t's true normals are its speculative ones [first[t], lim[t]),
  // the first of which starts at raw position fpos[t]
  std::vector<uint64_t> first(T, 0), lim(T, 0), fpos(T, 0);
  for (int t = 0; t + 1 < T; ++t) {
    const auto& hd = ch[t + 1].head;
    bool found = false;
    for (const auto& e : ch[t].tail) {
      auto it = std::lower_bound(hd.begin(), hd.end(), std::make_pair(e.first, (uint64_t)0));
      if (it != hd.end() && it->first == e.first) {
        lim[t] = e.second;
        first[t + 1] = it->second;
        fpos[t + 1] = e.first;
        found = true;
        break;
      }
    }
    if (!found) return -2;
  }
  lim[T - 1] = ch[T - 1].nspec;
  std::vector<uint64_t> off(T + 1, 0);
  for (int t = 0; t < T; ++t) off[t + 1] = off[t] + (lim[t] > first[t] ? lim[t] - first[t] : 0);
  if (off[T] < count) return -2;
  // pass 2: every chunk writes its true normals at its final offset
  std::vector<uint64_t> endpos(T, 0);
  {
    std::vector<std::thread> th;
    for (int t = 0; t < T; ++t) {
      if (off[t] >= count) break;
      const uint64_t n = std::min<uint64_t>(off[t + 1] - off[t], count - off[t]);
      th.emplace_back([&, t, n]() { endpos[t] = fill(out + off[t], n, fpos[t], s0, inc); });
    }
    for (auto& x : th) x.join();
  }
  int tc = 0;
  while (off[tc + 1] < count) ++tc;  // chunk holding normal count - 1
  *consumed = endpos[tc];
  return 0;
}

}  // extern "C"
