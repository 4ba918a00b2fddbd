// host_common.hpp -- host-side precision model and errors of the B200 solver.
//
// Restates the reference's configuration surface on the host:
//   PrecisionKind / EmulationMode / ArrayClass   precision.hpp:31-66
//   resolve_preset                               precision.cpp:58-88
//   PrecisionConfig::resolve                     precision.cpp:46-56
//   split_preset                                 physics.cpp:19-43
//   round_to                                     precision.hpp:167-174
#pragma once

#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>

namespace mpfd_b200 {

struct ConfigError : std::runtime_error {
    explicit ConfigError(const std::string& w) : std::runtime_error(w) {}
};
struct DeviceError : std::runtime_error {
    explicit DeviceError(const std::string& w) : std::runtime_error(w) {}
};

enum Kind : int { B16 = 0, B32 = 1, B64 = 2 };

inline int byte_width(int k) { return k == B16 ? 2 : (k == B32 ? 4 : 8); }

// RNE binary64 -> binary16 bit pattern, single rounding (integer formulation)
inline uint16_t half_bits(double x) {
    uint64_t b;
    std::memcpy(&b, &x, 8);
    const uint16_t sign = (uint16_t)((b >> 48) & 0x8000u);
    const uint64_t a = b & 0x7FFFFFFFFFFFFFFFull;
    if (a >= 0x7FF0000000000000ull) return (uint16_t)(sign | (a == 0x7FF0000000000000ull ? 0x7C00u : 0x7E00u));
    const int e = (int)(a >> 52) - 1023;
    const uint64_t sig = (a & 0xFFFFFFFFFFFFFull) | (a >> 52 ? (1ull << 52) : 0);
    if (e > 15) return (uint16_t)(sign | 0x7C00u);
    // keep bits above the target quantum 2^(max(e,-14)-10)
    const int qe = (e < -14 ? -14 : e) - 10;
    const int shift = 52 - (e - qe);  // bits of sig below the quantum
    if (shift >= 64) return sign;
    uint64_t keep = sig >> shift;
    const uint64_t rest = sig & ((1ull << shift) - 1);
    const uint64_t halfq = 1ull << (shift - 1);
    if (rest > halfq || (rest == halfq && (keep & 1))) ++keep;
    // keep counts quanta of 2^qe; rebuild
    if (e < -14) return (uint16_t)(sign | keep);  // subnormal (keep==1024 -> min normal, correct)
    if (keep == 2048) {                           // carried into the next binade
        if (e + 1 > 15) return (uint16_t)(sign | 0x7C00u);
        return (uint16_t)(sign | ((e + 1 + 15) << 10));
    }
    return (uint16_t)(sign | ((e + 15) << 10) | (keep & 0x3FFu));
}

inline double half_value(uint16_t h) {
    const int e = (h >> 10) & 0x1F;
    const int m = h & 0x3FF;
    double v;
    if (e == 0) v = std::ldexp((double)m, -24);
    else if (e == 31) v = m ? NAN : INFINITY;
    else v = std::ldexp((double)(m | 0x400), e - 25);
    return (h & 0x8000u) ? -v : v;
}

inline double round_to(int kind, double x) {
    if (kind == B64) return x;
    if (kind == B32) return (double)(float)x;
    return half_value(half_bits(x));
}

inline int parse_kind(const std::string& s) {
    if (s == "B16") return B16;
    if (s == "B32") return B32;
    if (s == "B64") return B64;
    throw ConfigError("unknown precision kind '" + s + "' (expected B16, B32 or B64)");
}

struct Precision {
    int q = B64, rk = B64, res = B64, wk = B64;
    int emulation = 0;  // 0 strict, 1 storeround
    std::map<std::string, int> overrides;

    int resolve(int cls, const std::string& name) const {
        auto it = overrides.find(name);
        if (it != overrides.end()) return it->second;
        switch (cls) {
            case 0: return q;
            case 1: return rk;
            case 2: return res;
            case 3: return wk;
            default: return B64;
        }
    }
};

inline bool preset(const std::string& name, Precision& p) {
    struct P {
        const char* n;
        int q, rk, res, wk;
    };
    static const P table[] = {
        {"DP", B64, B64, B64, B64},      {"SP", B32, B32, B32, B32},
        {"HP", B16, B16, B16, B16},      {"SPDP", B64, B64, B32, B32},
        {"SPDP-wk", B64, B64, B64, B32}, {"SPDP-res", B64, B64, B32, B64},
        {"HPSP", B32, B32, B16, B16},    {"HPSP-wk", B32, B32, B32, B16},
        {"HPSP-res", B32, B32, B16, B32},
    };
    for (const auto& e : table)
        if (name == e.n) {
            p.q = e.q;
            p.rk = e.rk;
            p.res = e.res;
            p.wk = e.wk;
            return true;
        }
    return false;
}

inline bool split(const std::string& name, double w[7]) {
    for (int i = 0; i < 7; ++i) w[i] = 0.0;
    if (name == "Divergence") w[0] = 1.0;
    else if (name == "Feiereisen") w[0] = w[3] = w[6] = 0.5;
    else if (name == "Blaisdell") w[0] = w[2] = w[5] = 0.5;
    else if (name == "Kok") w[0] = w[1] = w[4] = 0.5;
    else if (name == "KGP")
        for (int i = 0; i < 7; ++i) w[i] = 0.25;
    else return false;
    return true;
}

// field names of make_solver_fields (physics.cpp:441-475)
static const char* const kQNames[5] = {"rho", "rhou", "rhov", "rhow", "rhoE"};
static const char* const kTNames[5] = {"rk_rho", "rk_rhou", "rk_rhov", "rk_rhow", "rk_rhoE"};
static const char* const kRNames[5] = {"res_rho", "res_rhou", "res_rhov", "res_rhow", "res_rhoE"};
static const char* const kPNames[5] = {"u", "v", "w", "p", "T"};
static const char* const kGNames[12] = {"dudx", "dudy", "dudz", "dvdx", "dvdy", "dvdz",
                                        "dwdx", "dwdy", "dwdz", "dTdx", "dTdy", "dTdz"};

}  // namespace mpfd_b200
