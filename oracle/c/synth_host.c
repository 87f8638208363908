/* TEST / BASELINE INFRASTRUCTURE (oracle/): the host twin of csrc/synth.cu.
 *
 * bench.py's CPU reference arm regenerates the GPU arm's synthetic expert
 * weights as float64 (the reference's dtype, model.py:173-186) without
 * loading libbmoe or touching a GPU. Same integer recipe as the kernel and
 * as paper_2511_10054_b200/synth.py (which the tests compare bit for bit):
 *   out[i] = lut64[(mix64(base + i/4) >> 16*(i%4)) & 0xFFFF]
 * The caller splits [0, n) into 4-aligned ranges and runs them on threads
 * (ctypes drops the GIL). Built by `make -C oracle` into oracle/_lib/. */
#include <stdint.h>

static inline uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

static inline float bits_f32(uint32_t u) {
    union { uint32_t u; float f; } x;
    x.u = u;
    return x.f;
}

static inline uint32_t f32_bits(float f) {
    union { uint32_t u; float f; } x;
    x.f = f;
    return x.u;
}

/* clustered experts: bf16_rn(b + spread * e) with b, e from the bf16 lut of
 * the base / delta matrices (fp32 ops, one rounding each), widened to f64 */
void synth_mix_f64_range(uint64_t base_key, uint64_t delta_key, float spread, int64_t n, int64_t start,
                         int64_t count, const uint16_t *lut16, double *out) {
    const int64_t end = start + count < n ? start + count : n;
    for (int64_t i = start; i < end; i += 4) {
        const uint64_t zb = mix64(base_key + (uint64_t)(i / 4)), zd = mix64(delta_key + (uint64_t)(i / 4));
        const int64_t m = end - i < 4 ? end - i : 4;
        for (int64_t j = 0; j < m; ++j) {
            const float b = bits_f32((uint32_t)lut16[(zb >> (16 * j)) & 0xFFFF] << 16);
            const float e = bits_f32((uint32_t)lut16[(zd >> (16 * j)) & 0xFFFF] << 16);
            const float prod = spread * e;
            const float v = b + prod;
            uint32_t u = f32_bits(v);
            u = (u + 0x7FFFu + ((u >> 16) & 1u)) & 0xFFFF0000u; /* round to nearest even bf16 */
            out[i - start + j] = (double)bits_f32(u);
        }
    }
}

/* values [start, start + count) of a matrix of n values; start % 4 == 0 */
void synth_f64_range(uint64_t base, int64_t n, int64_t start, int64_t count, const double *lut64, double *out) {
    const int64_t end = start + count < n ? start + count : n;
    for (int64_t i = start; i < end; i += 4) {
        const uint64_t z = mix64(base + (uint64_t)(i / 4));
        const int64_t m = end - i < 4 ? end - i : 4;
        for (int64_t j = 0; j < m; ++j) out[i - start + j] = lut64[(z >> (16 * j)) & 0xFFFF];
    }
}
