// hadamard.cpp -- Hadamard factor tables for the RHT.
//
// Reading R7: H_n = kron(H_b, H_{2^a}); H_{2^a} is Sylvester (computed on the
// fly in the kernels as (-1)^popcount(i & j)); H_b (b > 1) is the Paley-I matrix of order
// b = q + 1, q = 3 mod 4 a prime or 27 / 343:
//     H_b = I + S,  S[0][1..q] = +1,  S[1..q][0] = -1,  S[1+i][1+j] = chi(g_i - g_j),
// chi the quadratic character of GF(q), g_i the field element whose base-p digits are i.
// GF(27) = GF(3)[x]/(x^3 + 2x + 1), GF(343) = GF(7)[x]/(x^3 + 4).
// b is the smallest supported order for which n / b is a power of two.
#include <cstdio>
#include <map>
#include <mutex>
#include <vector>

#include "internal.h"

namespace qtip {
namespace {

constexpr int kMaxOrder = 1024;

bool prime(int q) {
    if (q < 2) return false;
    for (int d = 2; d * d <= q; ++d)
        if (q % d == 0) return false;
    return true;
}

}  // namespace
bool paley_field_supported(int q) { return q % 4 == 3 && (prime(q) || q == 27 || q == 343); }
namespace {

// GF(p^deg) with elements stored as their integer index sum_d c_d p^d.
struct Field {
    int p = 0, deg = 0, q = 0;
    int mod[3] = {0, 0, 0};   // x^3 = -(mod[2] x^2 + mod[1] x + mod[0])
    int sub(int u, int v) const {
        int r = 0, pw = 1;
        for (int d = 0; d < deg; ++d) {
            const int cu = (u / pw) % p, cv = (v / pw) % p;
            r += ((cu - cv + p) % p) * pw;
            pw *= p;
        }
        return r;
    }
    int mul(int u, int v) const {
        if (deg == 1) return (u * v) % p;
        int cu[3], cv[3], prod[5] = {0, 0, 0, 0, 0};
        for (int d = 0, pw = 1; d < 3; ++d, pw *= p) { cu[d] = (u / pw) % p; cv[d] = (v / pw) % p; }
        for (int i = 0; i < 3; ++i)
            for (int j = 0; j < 3; ++j) prod[i + j] += cu[i] * cv[j];
        for (int e = 4; e >= 3; --e) {
            const int t = prod[e] % p;
            prod[e] = 0;
            for (int d = 0; d < 3; ++d) prod[e - 3 + d] -= t * mod[d];
        }
        int r = 0;
        for (int d = 2; d >= 0; --d) r = r * p + (((prod[d] % p) + p) % p);
        return r;
    }
};

Field make_field(int q) {
    Field f;
    f.q = q;
    if (prime(q)) { f.p = q; f.deg = 1; }
    else if (q == 27) { f.p = 3; f.deg = 3; f.mod[0] = 1; f.mod[1] = 2; f.mod[2] = 0; }
    else { f.p = 7; f.deg = 3; f.mod[0] = 4; f.mod[1] = 0; f.mod[2] = 0; }
    return f;
}

// +1 / -1 entries of the Paley-I matrix, row-major.
std::vector<int8_t> paley(int b) {
    const int q = b - 1;
    const Field F = make_field(q);
    std::vector<char> is_sq(q, 0);
    for (int e = 1; e < q; ++e) is_sq[F.mul(e, e)] = 1;
    std::vector<int8_t> H((size_t)b * b, 0);
    for (int i = 0; i < b; ++i) H[(size_t)i * b + i] = 1;
    for (int j = 1; j < b; ++j) H[j] += 1;                       // S[0][j] = +1
    for (int i = 1; i < b; ++i) H[(size_t)i * b] += -1;          // S[i][0] = -1
    for (int i = 0; i < q; ++i)
        for (int j = 0; j < q; ++j) {
            if (i == j) continue;                                // chi(0) = 0
            const int d = F.sub(i, j);
            H[(size_t)(i + 1) * b + (j + 1)] += is_sq[d] ? 1 : -1;
        }
    return H;
}

std::mutex g_mu;
std::map<std::pair<int, int>, uint32_t*> g_tables;   // (device, b) -> device bits

}  // namespace

bool hadamard_factor(int64_t n, int* b, int* a) {
    if (n <= 0) return false;
    for (int cand = 1; cand <= kMaxOrder; ++cand) {
        if (cand > 1 && !paley_field_supported(cand - 1)) continue;
        if (n % cand) continue;
        const int64_t r = n / cand;
        if ((r & (r - 1)) == 0) {
            int e = 0;
            while ((int64_t(1) << e) < r) ++e;
            *b = cand;
            *a = e;
            return true;
        }
    }
    return false;
}

const uint32_t* hadamard_table_device(int b, bool transpose, cudaError_t* err) {
    int dev = 0;
    *err = cudaGetDevice(&dev);
    if (*err != cudaSuccess) return nullptr;
    std::lock_guard<std::mutex> lock(g_mu);
    const int key = transpose ? -b : b;
    auto it = g_tables.find({dev, key});
    if (it != g_tables.end()) return it->second;
    const std::vector<int8_t> H = paley(b);
    const int wpr = (b + 31) / 32;                                  // words per bit row
    std::vector<uint32_t> bits((size_t)b * wpr, 0u);
    for (int i = 0; i < b; ++i)
        for (int j = 0; j < b; ++j) {
            const int8_t h = transpose ? H[(size_t)j * b + i] : H[(size_t)i * b + j];
            if (h < 0) bits[(size_t)i * wpr + (j >> 5)] |= 1u << (j & 31);
        }
    uint32_t* d = nullptr;
    *err = cudaMalloc(&d, bits.size() * sizeof(uint32_t));
    if (*err != cudaSuccess) return nullptr;
    *err = cudaMemcpy(d, bits.data(), bits.size() * sizeof(uint32_t), cudaMemcpyHostToDevice);
    if (*err != cudaSuccess) { cudaFree(d); return nullptr; }
    g_tables[{dev, key}] = d;
    return d;
}

}  // namespace qtip

extern "C" int qtip_internal_paley_host(int b, int8_t* out) {
    // Test hook: host copy of the library's own H_b (b x b, +1/-1), for orthogonality checks.
    if (b < 2 || !qtip::paley_field_supported(b - 1)) return -1;
    const std::vector<int8_t> H = qtip::paley(b);
    for (size_t i = 0; i < H.size(); ++i) out[i] = H[i];
    return 0;
}
