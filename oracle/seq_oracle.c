/*
 * seq_oracle.c — sequential topological oracle over the interval CSR.
 * TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
 *
 * Restates, in plain C, the "sequential topological execution oracle"
 * for the token definition of oracle/tokens.py: nodes are
 * executed one at a time in a topological order; each folds its
 * predecessors' 32-bit terms term(u) = mix64(tok[u] ^ mix64(u + G3)) >> 32
 * into an exact sum (SPEC.md:530-531 fold, builder definition).  It shares no code with the CUDA executor and is an
 * independent restatement of oracle/taskbench_np.py.
 *
 * Build: oracle/Makefile  ->  oracle/_build/liboracle.so
 */
#include <stdint.h>
#include <stdlib.h>

#define G1 0x9E3779B97F4A7C15ull
#define G2 0xD1B54A32D192ED03ull
#define G3 0x8CB92BA72F3D8DD7ull
#define LCG_A 6364136223846793005ull
#define LCG_C 1442695040888963407ull

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

/* LCG^n as an affine map (A, C): binary exponentiation of composition. */
static void affine_pow(uint32_t n, uint64_t* A, uint64_t* Cc) {
  uint64_t ra = 1, rc = 0, ba = LCG_A, bc = LCG_C;
  while (n) {
    if (n & 1u) { rc = ba * rc + bc; ra = ba * ra; }
    bc = ba * bc + bc;
    ba = ba * ba;
    n >>= 1;
  }
  *A = ra;
  *Cc = rc;
}

/* The literal loop, for the timed CPU run of COMPUTE bodies. */
uint64_t td_oracle_compute_loop(uint64_t h, uint32_t iters) {
  uint64_t r = 0;
  for (int l = 0; l < 64; ++l) {
    uint64_t x = mix64(h ^ ((uint64_t)(l + 1) * G2));
    for (uint32_t i = 0; i < iters; ++i) x = LCG_A * x + LCG_C;
    r ^= x;
  }
  return r;
}

/*
 * Returns 0 on success, -1 on a bad order (a predecessor not yet executed),
 * -2 on a bad interval.  order == NULL means id order.  literal_loop != 0 runs
 * COMPUTE bodies with the real loop instead of the affine shortcut.
 */
int td_oracle_run(int64_t n, const int64_t* pred_ptr, const int32_t* pred_iv,
                  const uint8_t* kind, const uint32_t* arg, const int64_t* order,
                  uint64_t seed, int literal_loop, const uint64_t* body_extra, uint64_t* tok) {
  uint8_t* done = (uint8_t*)calloc((size_t)(n > 0 ? n : 1), 1);
  if (!done) return -3;
  uint32_t cached_n = 0xFFFFFFFFu;
  uint64_t cA = 1, cC = 0;
  int rc = 0;
  for (int64_t i = 0; i < n && rc == 0; ++i) {
    const int64_t v = order ? order[i] : i;
    uint64_t acc = 0;
    for (int64_t k = pred_ptr[v]; k < pred_ptr[v + 1]; ++k) {
      const int32_t lo = pred_iv[2 * k], hi = pred_iv[2 * k + 1];
      if (lo < 0 || hi < lo || hi >= n) { rc = -2; break; }
      for (int32_t u = lo; u <= hi; ++u) {
        if (!done[u]) { rc = -1; break; }
        acc += mix64(tok[u] ^ mix64((uint64_t)u + G3)) >> 32;
      }
      if (rc) break;
    }
    if (rc) break;
    const uint64_t h0 = mix64(seed ^ mix64((uint64_t)v + G1));
    const uint64_t h = mix64(h0 ^ acc);
    uint64_t r = 0;
    if (kind && kind[v] == 2) {
      const uint32_t it = arg ? arg[v] : 0;
      if (literal_loop) {
        r = td_oracle_compute_loop(h, it);
      } else {
        if (it != cached_n) { affine_pow(it, &cA, &cC); cached_n = it; }
        for (int l = 0; l < 64; ++l) r ^= cA * mix64(h ^ ((uint64_t)(l + 1) * G2)) + cC;
      }
    }
    if (kind && kind[v] == 6) {  /* MEMORY(n): r = XOR_{k<n} (h + k*G2) */
      const uint32_t nw = arg ? arg[v] : 0;
      for (uint32_t k = 0; k < nw; ++k) r ^= h + (uint64_t)k * G2;
    }
    if (body_extra) r ^= body_extra[v];  /* STENCIL2D tile folds (td_oracle_stencil2d) */
    tok[v] = h ^ r;
    done[v] = 1;
  }
  free(done);
  return rc;
}

/*
 * Config-5 mini-app restated sequentially (BASELINE configs[4]): a u32 grid
 * nx x ny, 5-point update out = 2c + up + down + left + right (mod 2^32,
 * outside cells = 0), step 0 initialises cell (y, x) to
 * (uint32)mix64(seed ^ (y*nx + x + G2)).  Writes the per-task body result
 * r[t*ntiles + tile] = sum_k out_k * (2k+1) (k = row-major index inside the
 * 64x64 tile) and the final grid.  Returns 0 or -1 on bad sizes / -3 on OOM.
 */
int td_oracle_stencil2d(int32_t nx, int32_t ny, int32_t steps, uint64_t seed, uint64_t* r, uint32_t* final_grid) {
  const int T = 64;
  if (nx % T || ny % T || steps < 1) return -1;
  const int tx_n = nx / T, ty_n = ny / T;
  const int64_t nt = (int64_t)tx_n * ty_n;
  uint32_t* a = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nx * ny);
  uint32_t* b = (uint32_t*)malloc(sizeof(uint32_t) * (size_t)nx * ny);
  if (!a || !b) { free(a); free(b); return -3; }
  for (int64_t y = 0; y < ny; ++y)
    for (int64_t x = 0; x < nx; ++x) a[y * nx + x] = (uint32_t)mix64(seed ^ ((uint64_t)(y * nx + x) + G2));
  for (int step = 0; step < steps; ++step) {
    uint32_t* out = a;
    if (step > 0) {
      for (int64_t y = 0; y < ny; ++y)
        for (int64_t x = 0; x < nx; ++x) {
          const uint32_t c = a[y * nx + x];
          const uint32_t up = y > 0 ? a[(y - 1) * nx + x] : 0u, dn = y + 1 < ny ? a[(y + 1) * nx + x] : 0u;
          const uint32_t lf = x > 0 ? a[y * nx + x - 1] : 0u, rt = x + 1 < nx ? a[y * nx + x + 1] : 0u;
          b[y * nx + x] = 2u * c + up + dn + lf + rt;
        }
      uint32_t* tmp = a; a = b; b = tmp;
      out = a;
    }
    for (int64_t ty = 0; ty < ty_n; ++ty)
      for (int64_t tx = 0; tx < tx_n; ++tx) {
        uint64_t acc = 0;
        for (int y = 0; y < T; ++y)
          for (int x = 0; x < T; ++x) {
            const uint64_t k = (uint64_t)(y * T + x);
            acc += (uint64_t)out[(ty * T + y) * nx + tx * T + x] * (2 * k + 1);
          }
        r[step * nt + ty * tx_n + tx] = acc;
      }
  }
  if (final_grid)
    for (int64_t i = 0; i < (int64_t)nx * ny; ++i) final_grid[i] = a[i];
  free(a);
  free(b);
  return 0;
}
