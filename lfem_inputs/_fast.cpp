// Fast paths for lfem_inputs (input generation only; no assembly arithmetic).
// Same algorithms as the numpy reference implementations in __init__.py,
// which the tests compare against bit for bit.
#include <cstdint>
#include <cmath>

extern "C" {

// Skilling's transpose algorithm, 3-D, `bits` bits per axis (<= 21).
void lfin_hilbert_keys(int64_t n, const double* pts, const double* lo, const double* hi,
                       int bits, uint64_t* keys) {
    double span[3];
    for (int i = 0; i < 3; ++i) span[i] = (hi[i] > lo[i]) ? (hi[i] - lo[i]) : 1.0;
    const double scale = (double)((1u << bits) - 1);
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n; ++p) {
        uint32_t X[3];
        for (int i = 0; i < 3; ++i) {
            double q = std::floor((pts[3 * p + i] - lo[i]) / span[i] * scale + 0.5);
            if (q < 0) q = 0;
            if (q > scale) q = scale;
            X[i] = (uint32_t)q;
        }
        const uint32_t M = 1u << (bits - 1);
        for (uint32_t Q = M; Q > 1; Q >>= 1) {
            const uint32_t P = Q - 1;
            for (int i = 0; i < 3; ++i) {
                if (X[i] & Q) {
                    X[0] ^= P;
                } else {
                    uint32_t t = (X[0] ^ X[i]) & P;
                    X[0] ^= t;
                    X[i] ^= t;
                }
            }
        }
        X[1] ^= X[0];
        X[2] ^= X[1];
        uint32_t t = 0;
        for (uint32_t Q = M; Q > 1; Q >>= 1)
            if (X[2] & Q) t ^= Q - 1;
        for (int i = 0; i < 3; ++i) X[i] ^= t;
        uint64_t key = 0;
        for (int b = bits - 1; b >= 0; --b)
            for (int i = 0; i < 3; ++i) key = (key << 1) | ((X[i] >> b) & 1u);
        keys[p] = key;
    }
}

// u(x) = sum_{l<=lmax, m} coef[l*l+l+m] Y_lm(x / |x|)  (real orthonormal,
// no Condon-Shortley phase; identical recursion to lfem_inputs.real_sh).
void lfin_sh_field(int64_t n, const double* xyz, int lmax, const double* coef,
                   const double* norms /* (lmax+1)^2: N_lm incl. sqrt2 for m != 0 */,
                   int normalize, double* out) {
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < n; ++p) {
        double x = xyz[3 * p], y = xyz[3 * p + 1], z = xyz[3 * p + 2];
        if (normalize) {
            double r = std::sqrt(x * x + y * y + z * z);
            x /= r; y /= r; z /= r;
        }
        double cm[16], sm[16];
        cm[0] = 1.0; sm[0] = 0.0;
        for (int m = 1; m <= lmax; ++m) {
            cm[m] = cm[m - 1] * x - sm[m - 1] * y;
            sm[m] = cm[m - 1] * y + sm[m - 1] * x;
        }
        double acc = 0.0;
        for (int m = 0; m <= lmax; ++m) {
            double dfact = 1.0;
            for (int k = 1; k < 2 * m; k += 2) dfact *= k;
            double qp2 = 0.0, qp = dfact, q = dfact;
            for (int l = m; l <= lmax; ++l) {
                if (l == m) {
                    q = qp;
                } else if (l == m + 1) {
                    q = z * (2 * m + 1) * qp;
                    qp2 = qp; qp = q;
                } else {
                    q = ((2 * l - 1) * z * qp - (l + m - 1) * qp2) / (l - m);
                    qp2 = qp; qp = q;
                }
                if (m == 0) {
                    acc += coef[l * l + l] * (norms[l * l + l] * q);
                } else {
                    acc += coef[l * l + l + m] * (norms[l * l + l + m] * q * cm[m]);
                    acc += coef[l * l + l - m] * (norms[l * l + l - m] * q * sm[m]);
                }
            }
        }
        out[p] = acc;
    }
}

}  // extern "C"
