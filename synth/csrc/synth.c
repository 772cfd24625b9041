/* synth.c — C rendering of the seeded input generator (synth/__init__.py).
 *
 * Test/bench infrastructure, NOT part of the method: it only draws the
 * synthetic checkpoint / adapter / prompt of SURVEY.md §8(c) O0 fast enough to
 * fill the multi-GB pinned pools of the 7B/13B configs.  Must be bit-identical
 * with the numpy rendering (tests/test_synth.py hash manifest).
 *
 * Build: gcc -O3 -ffp-contract=off -fPIC -shared -pthread (the x line below is
 * one IEEE multiply; contraction into an FMA would change the rounding).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <string.h>

static inline uint64_t splitmix64(uint64_t x) {
  uint64_t z = x + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

static inline uint16_t bf16_rne(float f) {
  uint32_t b;
  memcpy(&b, &f, 4);
  return (uint16_t)((b + 0x7FFFu + ((b >> 16) & 1u)) >> 16);
}

uint64_t synth_stream_key(uint64_t ns, uint64_t seed, uint64_t idx) {
  return splitmix64((ns << 56) ^ (seed << 24) ^ idx);
}

typedef struct {
  uint64_t key;
  float c;
  int is_norm;
  uint64_t cols_full, row0, col0, ncols;
  uint64_t r_begin, r_end;
  uint16_t* out;
} job_t;

static void run_rows(const job_t* j) {
  for (uint64_t r = j->r_begin; r < j->r_end; ++r) {
    uint64_t e0 = (j->row0 + r) * j->cols_full + j->col0;
    uint16_t* o = j->out + r * j->ncols;
    for (uint64_t c = 0; c < j->ncols; ++c) {
      uint64_t u = splitmix64(j->key + e0 + c);
      float x = ((float)(u >> 40) * 0x1p-23f - 1.0f) * j->c;
      if (j->is_norm) x = 1.0f + x;
      o[c] = bf16_rne(x);
    }
  }
}

static void* thread_main(void* p) {
  run_rows((const job_t*)p);
  return NULL;
}

/* Fill out[nrows x ncols] (row-major, bf16 bits) with the sub-block
 * [row0, row0+nrows) x [col0, col0+ncols) of the unsharded tensor whose row
 * length is cols_full (element index e = row*cols_full + col).  1-D tensors
 * use rows_full = 1.  Returns 0 on success. */
int synth_fill_bf16(uint64_t ns, uint64_t seed, uint64_t idx, double sigma, int is_norm,
                    uint64_t cols_full, uint64_t row0, uint64_t nrows, uint64_t col0,
                    uint64_t ncols, uint16_t* out, int nthreads) {
  if (nthreads < 1) nthreads = 1;
  if (nthreads > 256) nthreads = 256;
  job_t base;
  base.key = synth_stream_key(ns, seed, idx);
  base.c = (float)(sigma * sqrt(3.0));
  base.is_norm = is_norm;
  base.cols_full = cols_full;
  base.row0 = row0;
  base.col0 = col0;
  base.ncols = ncols;
  base.out = out;
  if (nthreads == 1 || nrows * ncols < (1u << 20)) {
    base.r_begin = 0;
    base.r_end = nrows;
    run_rows(&base);
    return 0;
  }
  if ((uint64_t)nthreads > nrows) nthreads = (int)nrows;
  pthread_t th[256];
  job_t jobs[256];
  int created[256];
  uint64_t per = (nrows + nthreads - 1) / nthreads;
  for (int t = 0; t < nthreads; ++t) {
    jobs[t] = base;
    jobs[t].r_begin = per * t < nrows ? per * t : nrows;
    jobs[t].r_end = per * (t + 1) < nrows ? per * (t + 1) : nrows;
    created[t] = pthread_create(&th[t], NULL, thread_main, &jobs[t]) == 0;
    if (!created[t]) run_rows(&jobs[t]);
  }
  for (int t = 0; t < nthreads; ++t)
    if (created[t]) pthread_join(th[t], NULL);
  return 0;
}

/* tok_i = splitmix64(key(2, seed, 0) + i) mod V */
void synth_prompt(uint64_t seed, uint64_t vocab, uint64_t n, int32_t* out) {
  uint64_t key = synth_stream_key(2, seed, 0);
  for (uint64_t i = 0; i < n; ++i) out[i] = (int32_t)(splitmix64(key + i) % vocab);
}
