// glibc_math.cuh -- bit-exact erf and exp, host and device.
//
// The reference builds its generator columns with std::erf (gaussian_moment_vector,
// newton.hpp:21-37) and std::exp (gaussian_sample_vector, newton.hpp:43-52), i.e. with the
// host's glibc (2.39 in this image, x86-64). CUDA's own erf/exp are faithfully rounded but
// differ from glibc in the last bit for a few percent of arguments, and the erf-difference
// cell integral erf(t*x_{i+1}) - erf(t*x_i) amplifies a one-ulp difference by up to len
// (SURVEY §0.4). So the generator evaluates the SAME algorithms glibc runs, operation for
// operation, and its columns are bit-identical to the reference's.
//
// * erf: the fdlibm s_erf.c algorithm (Sun Microsystems, 1993; coefficients published with
//   it), in the operation order of glibc 2.39's x86-64 build of erf, which uses no FMA:
//   four argument ranges with rational approximations, and for 1.25 <= |x| < 6 the product
//   exp(-z*z - 0.5625) * exp((z-|x|)*(z+|x|) + R/S) with z = |x| truncated to its high word.
// * exp: the 2018 table-driven exp (EXP_TABLE_BITS = 7, degree-5 polynomial) that glibc
//   selects through its ifunc on a host with FMA + AVX2 (__exp_fma): exp(x) = 2^(k/128) *
//   exp(r), |r| <= ln2/256, with the FMA placement of that build. The 2^(i/128) table below
//   follows its construction (tab[2i+1] = bits(2^(i/128)) - (i << 45), tab[2i] = bits of
//   the rounding tail); tools/glibc_math/dump_libm_consts.py confirms every entry and every
//   coefficient against the installed libm.so.6.
//
// Every arithmetic step is an explicit round-to-nearest intrinsic (device) or an operation
// in a translation unit compiled with -ffp-contract=off (host), so no compiler may contract
// or reassociate it. tools/glibc_math/check_vs_libm.cpp compares the host instantiation with
// libm bit for bit over 1e8+ arguments; tests/test_gpu_parity.py compares the device one.
#pragma once

#include <cstdint>
#include <cstring>

#if defined(__CUDACC__)
#define LS_GM_HD __host__ __device__ __forceinline__
#else
#include <cmath>
#define LS_GM_HD inline
#endif

namespace ls {
namespace gm {

// 2^(i/128) table of the table-driven exp: {tail_i, bits(2^(i/128)) - (i << 45)} per i.
#define LS_GM_EXP_TABLE_INIT \
    0x0000000000000000ULL, 0x3ff0000000000000ULL, 0x3c9b3b4f1a88bf6eULL, 0x3feff63da9fb3335ULL, \
    0xbc7160139cd8dc5dULL, 0x3fefec9a3e778061ULL, 0xbc905e7a108766d1ULL, 0x3fefe315e86e7f85ULL, \
    0x3c8cd2523567f613ULL, 0x3fefd9b0d3158574ULL, 0xbc8bce8023f98efaULL, 0x3fefd06b29ddf6deULL, \
    0x3c60f74e61e6c861ULL, 0x3fefc74518759bc8ULL, 0x3c90a3e45b33d399ULL, 0x3fefbe3ecac6f383ULL, \
    0x3c979aa65d837b6dULL, 0x3fefb5586cf9890fULL, 0x3c8eb51a92fdeffcULL, 0x3fefac922b7247f7ULL, \
    0x3c3ebe3d702f9cd1ULL, 0x3fefa3ec32d3d1a2ULL, 0xbc6a033489906e0bULL, 0x3fef9b66affed31bULL, \
    0xbc9556522a2fbd0eULL, 0x3fef9301d0125b51ULL, 0xbc5080ef8c4eea55ULL, 0x3fef8abdc06c31ccULL, \
    0xbc91c923b9d5f416ULL, 0x3fef829aaea92de0ULL, 0x3c80d3e3e95c55afULL, 0x3fef7a98c8a58e51ULL, \
    0xbc801b15eaa59348ULL, 0x3fef72b83c7d517bULL, 0xbc8f1ff055de323dULL, 0x3fef6af9388c8deaULL, \
    0x3c8b898c3f1353bfULL, 0x3fef635beb6fcb75ULL, 0xbc96d99c7611eb26ULL, 0x3fef5be084045cd4ULL, \
    0x3c9aecf73e3a2f60ULL, 0x3fef54873168b9aaULL, 0xbc8fe782cb86389dULL, 0x3fef4d5022fcd91dULL, \
    0x3c8a6f4144a6c38dULL, 0x3fef463b88628cd6ULL, 0x3c807a05b0e4047dULL, 0x3fef3f49917ddc96ULL, \
    0x3c968efde3a8a894ULL, 0x3fef387a6e756238ULL, 0x3c875e18f274487dULL, 0x3fef31ce4fb2a63fULL, \
    0x3c80472b981fe7f2ULL, 0x3fef2b4565e27cddULL, 0xbc96b87b3f71085eULL, 0x3fef24dfe1f56381ULL, \
    0x3c82f7e16d09ab31ULL, 0x3fef1e9df51fdee1ULL, 0xbc3d219b1a6fbffaULL, 0x3fef187fd0dad990ULL, \
    0x3c8b3782720c0ab4ULL, 0x3fef1285a6e4030bULL, 0x3c6e149289cecb8fULL, 0x3fef0cafa93e2f56ULL, \
    0x3c834d754db0abb6ULL, 0x3fef06fe0a31b715ULL, 0x3c864201e2ac744cULL, 0x3fef0170fc4cd831ULL, \
    0x3c8fdd395dd3f84aULL, 0x3feefc08b26416ffULL, 0xbc86a3803b8e5b04ULL, 0x3feef6c55f929ff1ULL, \
    0xbc924aedcc4b5068ULL, 0x3feef1a7373aa9cbULL, 0xbc9907f81b512d8eULL, 0x3feeecae6d05d866ULL, \
    0xbc71d1e83e9436d2ULL, 0x3feee7db34e59ff7ULL, 0xbc991919b3ce1b15ULL, 0x3feee32dc313a8e5ULL, \
    0x3c859f48a72a4c6dULL, 0x3feedea64c123422ULL, 0xbc9312607a28698aULL, 0x3feeda4504ac801cULL, \
    0xbc58a78f4817895bULL, 0x3feed60a21f72e2aULL, 0xbc7c2c9b67499a1bULL, 0x3feed1f5d950a897ULL, \
    0x3c4363ed60c2ac11ULL, 0x3feece086061892dULL, 0x3c9666093b0664efULL, 0x3feeca41ed1d0057ULL, \
    0x3c6ecce1daa10379ULL, 0x3feec6a2b5c13cd0ULL, 0x3c93ff8e3f0f1230ULL, 0x3feec32af0d7d3deULL, \
    0x3c7690cebb7aafb0ULL, 0x3feebfdad5362a27ULL, 0x3c931dbdeb54e077ULL, 0x3feebcb299fddd0dULL, \
    0xbc8f94340071a38eULL, 0x3feeb9b2769d2ca7ULL, 0xbc87deccdc93a349ULL, 0x3feeb6daa2cf6642ULL, \
    0xbc78dec6bd0f385fULL, 0x3feeb42b569d4f82ULL, 0xbc861246ec7b5cf6ULL, 0x3feeb1a4ca5d920fULL, \
    0x3c93350518fdd78eULL, 0x3feeaf4736b527daULL, 0x3c7b98b72f8a9b05ULL, 0x3feead12d497c7fdULL, \
    0x3c9063e1e21c5409ULL, 0x3feeab07dd485429ULL, 0x3c34c7855019c6eaULL, 0x3feea9268a5946b7ULL, \
    0x3c9432e62b64c035ULL, 0x3feea76f15ad2148ULL, 0xbc8ce44a6199769fULL, 0x3feea5e1b976dc09ULL, \
    0xbc8c33c53bef4da8ULL, 0x3feea47eb03a5585ULL, 0xbc845378892be9aeULL, 0x3feea34634ccc320ULL, \
    0xbc93cedd78565858ULL, 0x3feea23882552225ULL, 0x3c5710aa807e1964ULL, 0x3feea155d44ca973ULL, \
    0xbc93b3efbf5e2228ULL, 0x3feea09e667f3bcdULL, 0xbc6a12ad8734b982ULL, 0x3feea012750bdabfULL, \
    0xbc6367efb86da9eeULL, 0x3fee9fb23c651a2fULL, 0xbc80dc3d54e08851ULL, 0x3fee9f7df9519484ULL, \
    0xbc781f647e5a3ecfULL, 0x3fee9f75e8ec5f74ULL, 0xbc86ee4ac08b7db0ULL, 0x3fee9f9a48a58174ULL, \
    0xbc8619321e55e68aULL, 0x3fee9feb564267c9ULL, 0x3c909ccb5e09d4d3ULL, 0x3feea0694fde5d3fULL, \
    0xbc7b32dcb94da51dULL, 0x3feea11473eb0187ULL, 0x3c94ecfd5467c06bULL, 0x3feea1ed0130c132ULL, \
    0x3c65ebe1abd66c55ULL, 0x3feea2f336cf4e62ULL, 0xbc88a1c52fb3cf42ULL, 0x3feea427543e1a12ULL, \
    0xbc9369b6f13b3734ULL, 0x3feea589994cce13ULL, 0xbc805e843a19ff1eULL, 0x3feea71a4623c7adULL, \
    0xbc94d450d872576eULL, 0x3feea8d99b4492edULL, 0x3c90ad675b0e8a00ULL, 0x3feeaac7d98a6699ULL, \
    0x3c8db72fc1f0eab4ULL, 0x3feeace5422aa0dbULL, 0xbc65b6609cc5e7ffULL, 0x3feeaf3216b5448cULL, \
    0x3c7bf68359f35f44ULL, 0x3feeb1ae99157736ULL, 0xbc93091fa71e3d83ULL, 0x3feeb45b0b91ffc6ULL, \
    0xbc5da9b88b6c1e29ULL, 0x3feeb737b0cdc5e5ULL, 0xbc6c23f97c90b959ULL, 0x3feeba44cbc8520fULL, \
    0xbc92434322f4f9aaULL, 0x3feebd829fde4e50ULL, 0xbc85ca6cd7668e4bULL, 0x3feec0f170ca07baULL, \
    0x3c71affc2b91ce27ULL, 0x3feec49182a3f090ULL, 0x3c6dd235e10a73bbULL, 0x3feec86319e32323ULL, \
    0xbc87c50422622263ULL, 0x3feecc667b5de565ULL, 0x3c8b1c86e3e231d5ULL, 0x3feed09bec4a2d33ULL, \
    0xbc91bbd1d3bcbb15ULL, 0x3feed503b23e255dULL, 0x3c90cc319cee31d2ULL, 0x3feed99e1330b358ULL, \
    0x3c8469846e735ab3ULL, 0x3feede6b5579fdbfULL, 0xbc82dfcd978e9db4ULL, 0x3feee36bbfd3f37aULL, \
    0x3c8c1a7792cb3387ULL, 0x3feee89f995ad3adULL, 0xbc907b8f4ad1d9faULL, 0x3feeee07298db666ULL, \
    0xbc55c3d956dcaebaULL, 0x3feef3a2b84f15fbULL, 0xbc90a40e3da6f640ULL, 0x3feef9728de5593aULL, \
    0xbc68d6f438ad9334ULL, 0x3feeff76f2fb5e47ULL, 0xbc91eee26b588a35ULL, 0x3fef05b030a1064aULL, \
    0x3c74ffd70a5fddcdULL, 0x3fef0c1e904bc1d2ULL, 0xbc91bdfbfa9298acULL, 0x3fef12c25bd71e09ULL, \
    0x3c736eae30af0cb3ULL, 0x3fef199bdd85529cULL, 0x3c8ee3325c9ffd94ULL, 0x3fef20ab5fffd07aULL, \
    0x3c84e08fd10959acULL, 0x3fef27f12e57d14bULL, 0x3c63cdaf384e1a67ULL, 0x3fef2f6d9406e7b5ULL, \
    0x3c676b2c6c921968ULL, 0x3fef3720dcef9069ULL, 0xbc808a1883ccb5d2ULL, 0x3fef3f0b555dc3faULL, \
    0xbc8fad5d3ffffa6fULL, 0x3fef472d4a07897cULL, 0xbc900dae3875a949ULL, 0x3fef4f87080d89f2ULL, \
    0x3c74a385a63d07a7ULL, 0x3fef5818dcfba487ULL, 0xbc82919e2040220fULL, 0x3fef60e316c98398ULL, \
    0x3c8e5a50d5c192acULL, 0x3fef69e603db3285ULL, 0x3c843a59ac016b4bULL, 0x3fef7321f301b460ULL, \
    0xbc82d52107b43e1fULL, 0x3fef7c97337b9b5fULL, 0xbc892ab93b470dc9ULL, 0x3fef864614f5a129ULL, \
    0x3c74b604603a88d3ULL, 0x3fef902ee78b3ff6ULL, 0x3c83c5ec519d7271ULL, 0x3fef9a51fbc74c83ULL, \
    0xbc8ff7128fd391f0ULL, 0x3fefa4afa2a490daULL, 0xbc8dae98e223747dULL, 0x3fefaf482d8e67f1ULL, \
    0x3c8ec3bc41aa2008ULL, 0x3fefba1bee615a27ULL, 0x3c842b94c3a9eb32ULL, 0x3fefc52b376bba97ULL, \
    0x3c8a64a931d185eeULL, 0x3fefd0765b6e4540ULL, 0xbc8e37bae43be3edULL, 0x3fefdbfdad9cbe14ULL, \
    0x3c77893b4d91cd9dULL, 0x3fefe7c1819e90d8ULL, 0x3c5305c14160cc89ULL, 0x3feff3c22b8f71f1ULL


#if defined(__CUDACC__)
static __device__ const uint64_t kExpTabDev[256] = {LS_GM_EXP_TABLE_INIT};
#endif
static const uint64_t kExpTabHost[256] = {LS_GM_EXP_TABLE_INIT};

LS_GM_HD uint64_t tab(int i) {
#if defined(__CUDA_ARCH__)
    return __ldg(reinterpret_cast<const unsigned long long*>(kExpTabDev) + i);
#else
    return kExpTabHost[i];
#endif
}

LS_GM_HD uint64_t bits(double x) {
#if defined(__CUDA_ARCH__)
    return static_cast<uint64_t>(__double_as_longlong(x));
#else
    uint64_t u;
    std::memcpy(&u, &x, 8);
    return u;
#endif
}
LS_GM_HD double dbl(uint64_t u) {
#if defined(__CUDA_ARCH__)
    return __longlong_as_double(static_cast<long long>(u));
#else
    double x;
    std::memcpy(&x, &u, 8);
    return x;
#endif
}

// One rounding each; never contracted.
#if defined(__CUDA_ARCH__)
LS_GM_HD double mul(double a, double b) { return __dmul_rn(a, b); }
LS_GM_HD double add(double a, double b) { return __dadd_rn(a, b); }
LS_GM_HD double sub(double a, double b) { return __dsub_rn(a, b); }
LS_GM_HD double div(double a, double b) { return __ddiv_rn(a, b); }
LS_GM_HD double fma(double a, double b, double c) { return __fma_rn(a, b, c); }
#else
LS_GM_HD double mul(double a, double b) { return a * b; }
LS_GM_HD double add(double a, double b) { return a + b; }
LS_GM_HD double sub(double a, double b) { return a - b; }
LS_GM_HD double div(double a, double b) { return a / b; }
LS_GM_HD double fma(double a, double b, double c) { return std::fma(a, b, c); }
#endif

// ---- exp ---------------------------------------------------------------------------------
// Reduction constants and polynomial of the table-driven exp.
constexpr uint64_t kInvLn2N = 0x40671547652b82feULL;    // 128/ln2
constexpr uint64_t kShift = 0x4338000000000000ULL;      // 0x1.8p52
constexpr uint64_t kNegLn2HiN = 0xbf762e42fefa0000ULL;  // -ln2/128, high part
constexpr uint64_t kNegLn2LoN = 0xbd0cf79abc9e3b3aULL;  // -ln2/128, low part
constexpr uint64_t kC2 = 0x3fdffffffffffdbdULL;
constexpr uint64_t kC3 = 0x3fc555555555543cULL;
constexpr uint64_t kC4 = 0x3fa55555cf172b91ULL;
constexpr uint64_t kC5 = 0x3f81111167a4d017ULL;

// Results whose scale 2^(k/128) leaves the normal range: k > 0 is rescaled by 2^1009; k < 0
// goes through 2^1022 with the subnormal rounding done once (hi/lo split below 1.0).
LS_GM_HD double exp_specialcase(double tmp, uint64_t sbits, uint64_t ki) {
    if ((ki & 0x80000000ULL) == 0) {
        const double scale = dbl(sbits - (1009ULL << 52));
        return mul(fma(scale, tmp, scale), dbl(0x7f00000000000000ULL));  // * 2^1009
    }
    const double scale = dbl(sbits + (1022ULL << 52));
    const double st = mul(tmp, scale);
    double y = add(scale, st);
    if (y < 1.0) {
        const double hi = add(y, 1.0);
        const double lo = add(sub(scale, y), st);
        double t = add(sub(1.0, hi), y);
        t = add(t, lo);
        t = add(t, hi);
        y = sub(t, 1.0);
        if (y == 0.0) y = 0.0;  // never -0
    }
    return mul(y, dbl(0x0010000000000000ULL));  // * 2^-1022
}

LS_GM_HD double exp(double x) {
    const uint64_t ix = bits(x);
    uint32_t abstop = static_cast<uint32_t>(ix >> 52) & 0x7ff;
    if (abstop - 0x3c9u > 0x3eu) {                       // |x| < 2^-54 or |x| >= 512
        if (static_cast<int32_t>(abstop - 0x3c9u) < 0) return add(x, 1.0);
        if (abstop >= 0x409u) {                          // |x| >= 1024
            if (ix == 0xfff0000000000000ULL) return 0.0;
            if (abstop == 0x7ffu) return add(x, 1.0);
            if (ix >> 63) return 0.0;                    // underflow
            return dbl(0x7ff0000000000000ULL);           // overflow
        }
        abstop = 0;                                      // large |x|: special-cased below
    }
    double kd = fma(x, dbl(kInvLn2N), dbl(kShift));
    const uint64_t ki = bits(kd);
    kd = sub(kd, dbl(kShift));
    double r = fma(kd, dbl(kNegLn2HiN), x);
    r = fma(kd, dbl(kNegLn2LoN), r);
    const int idx = static_cast<int>(2 * (ki & 127));
    const uint64_t top = ki << 45;
    const double tail_r = add(r, dbl(tab(idx)));
    const uint64_t sbits = tab(idx + 1) + top;
    const double p23 = fma(r, dbl(kC3), dbl(kC2));
    const double r2 = mul(r, r);
    const double p45 = fma(r, dbl(kC5), dbl(kC4));
    double tmp = fma(p23, r2, tail_r);
    tmp = fma(mul(r2, r2), p45, tmp);
    if (abstop == 0) return exp_specialcase(tmp, sbits, ki);
    const double scale = dbl(sbits);
    return fma(scale, tmp, scale);
}

// ---- erf ---------------------------------------------------------------------------------
// fdlibm s_erf.c coefficients, by their published names (bit patterns of glibc 2.39's copy).
constexpr uint64_t kPp0 = 0x3fc06eba8214db68ULL;  // 0.12837916709551256
constexpr uint64_t kPp1 = 0xbfd4cd7d691cb913ULL;  // -0.3250421072470015
constexpr uint64_t kPp2 = 0xbf9d2a51dbd7194fULL;  // -0.02848174957559851
constexpr uint64_t kPp3 = 0xbf77a291236668e4ULL;  // -0.005770270296489442
constexpr uint64_t kPp4 = 0xbef8ead6120016acULL;  // -2.3763016656650163e-05
constexpr uint64_t kQq1 = 0x3fd97779cddadc09ULL;  // 0.39791722395915535
constexpr uint64_t kQq2 = 0x3fb0a54c5536cebaULL;  // 0.0650222499887673
constexpr uint64_t kQq3 = 0x3f74d022c4d36b0fULL;  // 0.005081306281875766
constexpr uint64_t kQq4 = 0x3f215dc9221c1a10ULL;  // 0.00013249473800432164
constexpr uint64_t kQq5 = 0xbed09c4342a26120ULL;  // -3.960228278775368e-06
constexpr uint64_t kPa0 = 0xbf6359b8bef77538ULL;  // -0.0023621185607526594
constexpr uint64_t kPa1 = 0x3fda8d00ad92b34dULL;  // 0.41485611868374833
constexpr uint64_t kPa2 = 0xbfd7d240fbb8c3f1ULL;  // -0.3722078760357013
constexpr uint64_t kPa3 = 0x3fd45fca805120e4ULL;  // 0.31834661990116175
constexpr uint64_t kPa4 = 0xbfbc63983d3e28ecULL;  // -0.11089469428239668
constexpr uint64_t kPa5 = 0x3fa22a36599795ebULL;  // 0.035478304325618236
constexpr uint64_t kPa6 = 0xbf61bf380a96073fULL;  // -0.002166375594868791
constexpr uint64_t kQa1 = 0x3fbb3e6618eee323ULL;  // 0.10642088040084423
constexpr uint64_t kQa2 = 0x3fe14af092eb6f33ULL;  // 0.540397917702171
constexpr uint64_t kQa3 = 0x3fb2635cd99fe9a7ULL;  // 0.07182865441419627
constexpr uint64_t kQa4 = 0x3fc02660e763351fULL;  // 0.12617121980876164
constexpr uint64_t kQa5 = 0x3f8bedc26b51dd1cULL;  // 0.01363708391202905
constexpr uint64_t kQa6 = 0x3f888b545735151dULL;  // 0.011984499846799107
constexpr uint64_t kRa0 = 0xbf843412600d6435ULL;  // -0.009864944034847148
constexpr uint64_t kRa1 = 0xbfe63416e4ba7360ULL;  // -0.6938585727071818
constexpr uint64_t kRa2 = 0xc0251e0441b0e726ULL;  // -10.558626225323291
constexpr uint64_t kRa3 = 0xc04f300ae4cba38dULL;  // -62.375332450326006
constexpr uint64_t kRa4 = 0xc0644cb184282266ULL;  // -162.39666946257347
constexpr uint64_t kRa5 = 0xc067135cebccabb2ULL;  // -184.60509290671104
constexpr uint64_t kRa6 = 0xc054526557e4d2f2ULL;  // -81.2874355063066
constexpr uint64_t kRa7 = 0xc023a0efc69ac25cULL;  // -9.814329344169145
constexpr uint64_t kSa1 = 0x4033a6b9bd707687ULL;  // 19.651271667439257
constexpr uint64_t kSa2 = 0x4061350c526ae721ULL;  // 137.65775414351904
constexpr uint64_t kSa3 = 0x407b290dd58a1a71ULL;  // 434.56587747522923
constexpr uint64_t kSa4 = 0x40842b1921ec2868ULL;  // 645.3872717332679
constexpr uint64_t kSa5 = 0x407ad02157700314ULL;  // 429.00814002756783
constexpr uint64_t kSa6 = 0x405b28a3ee48ae2cULL;  // 108.63500554177944
constexpr uint64_t kSa7 = 0x401a47ef8e484a93ULL;  // 6.570249770319282
constexpr uint64_t kSa8 = 0xbfaeeff2ee749a62ULL;  // -0.0604244152148581
constexpr uint64_t kRb0 = 0xbf84341239e86f4aULL;  // -0.0098649429247001
constexpr uint64_t kRb1 = 0xbfe993ba70c285deULL;  // -0.799283237680523
constexpr uint64_t kRb2 = 0xc031c209555f995aULL;  // -17.757954917754752
constexpr uint64_t kRb3 = 0xc064145d43c5ed98ULL;  // -160.63638485582192
constexpr uint64_t kRb4 = 0xc083ec881375f228ULL;  // -637.5664433683896
constexpr uint64_t kRb5 = 0xc09004616a2e5992ULL;  // -1025.0951316110772
constexpr uint64_t kRb6 = 0xc07e384e9bdc383fULL;  // -483.5191916086514
constexpr uint64_t kSb1 = 0x403e568b261d5190ULL;  // 30.33806074348246
constexpr uint64_t kSb2 = 0x40745cae221b9f0aULL;  // 325.7925129965739
constexpr uint64_t kSb3 = 0x409802eb189d5118ULL;  // 1536.729586084437
constexpr uint64_t kSb4 = 0x40a8ffb7688c246aULL;  // 3199.8582195085955
constexpr uint64_t kSb5 = 0x40a3f219cedf3be6ULL;  // 2553.0504064331644
constexpr uint64_t kSb6 = 0x407da874e79fe763ULL;  // 474.52854120695537
constexpr uint64_t kSb7 = 0xc03670e242712d62ULL;  // -22.44095244658582
constexpr uint64_t kErx = 0x3feb0ac160000000ULL;  // 0.8450629115104675
constexpr uint64_t kEfx = 0x3fc06eba8214db69ULL;  // 0.1283791670955126
constexpr uint64_t kEfx16 = 0x40006eba8214db69ULL;  // 2.0540666735282014

// Polynomial evaluation order is that of glibc 2.39's x86-64 erf (no FMA), e.g. for |x| <
// 0.84375: r = ((pp2 + z*pp3)*z^2 + (pp0 + z*pp1)) + z^4*pp4.
LS_GM_HD double erf(double x) {
    const uint64_t ux = bits(x);
    const uint32_t hx = static_cast<uint32_t>(ux >> 32);
    const uint32_t ix = hx & 0x7fffffffu;
    const bool neg = (hx >> 31) != 0;
    if (ix >= 0x7ff00000u)  // erf(nan) = nan, erf(+-inf) = +-1
        return add(neg ? -1.0 : 1.0, div(1.0, x));
    if (ix < 0x3feb0000u) {  // |x| < 0.84375
        if (ix < 0x3e300000u) {  // |x| < 2^-28
            if ((hx & 0x7f800000u) == 0)  // avoid spurious underflow
                return mul(add(mul(x, 16.0), mul(x, dbl(kEfx16))), 0.0625);
            return add(mul(x, dbl(kEfx)), x);
        }
        const double z = mul(x, x);
        const double z2 = mul(z, z);
        const double z4 = mul(z2, z2);
        double r = add(mul(add(mul(dbl(kPp3), z), dbl(kPp2)), z2), add(mul(dbl(kPp1), z), dbl(kPp0)));
        r = add(r, mul(dbl(kPp4), z4));
        const double s1 = add(mul(add(mul(dbl(kQq3), z), dbl(kQq2)), z2), add(mul(dbl(kQq1), z), 1.0));
        const double s = add(mul(add(mul(z, dbl(kQq5)), dbl(kQq4)), z4), s1);
        return add(mul(div(r, s), x), x);
    }
    if (ix < 0x3ff40000u) {  // 0.84375 <= |x| < 1.25
        const double s = sub(dbl(ux & 0x7fffffffffffffffULL), 1.0);
        const double s2 = mul(s, s);
        const double s4 = mul(s2, s2);
        const double s6 = mul(s2, s4);
        double p = add(mul(add(mul(dbl(kPa3), s), dbl(kPa2)), s2), add(mul(dbl(kPa1), s), dbl(kPa0)));
        p = add(p, mul(add(mul(dbl(kPa5), s), dbl(kPa4)), s4));
        p = add(p, mul(dbl(kPa6), s6));
        double q = add(mul(add(mul(dbl(kQa3), s), dbl(kQa2)), s2), add(mul(dbl(kQa1), s), 1.0));
        q = add(q, mul(add(mul(s, dbl(kQa5)), dbl(kQa4)), s4));
        q = add(q, mul(s6, dbl(kQa6)));
        const double pq = div(p, q);
        return neg ? sub(-dbl(kErx), pq) : add(pq, dbl(kErx));
    }
    if (ix >= 0x40180000u)  // |x| >= 6: +-(1 - tiny)
        return neg ? -1.0 : 1.0;
    const double ax = dbl(ux & 0x7fffffffffffffffULL);
    const double s = div(1.0, mul(x, x));
    const double s2 = mul(s, s);
    const double s4 = mul(s2, s2);
    const double s6 = mul(s4, s2);
    double R, S;
    if (ix < 0x4006db6eu) {  // |x| < 1/0.35
        R = add(mul(add(mul(s, dbl(kRa3)), dbl(kRa2)), s2), add(mul(dbl(kRa1), s), dbl(kRa0)));
        R = add(R, mul(add(mul(dbl(kRa5), s), dbl(kRa4)), s4));
        R = add(R, mul(add(mul(dbl(kRa7), s), dbl(kRa6)), s6));
        double t = add(mul(s2, add(mul(dbl(kSa3), s), dbl(kSa2))), add(mul(dbl(kSa1), s), 1.0));
        t = add(t, mul(add(mul(dbl(kSa5), s), dbl(kSa4)), s4));
        S = add(mul(add(mul(s, dbl(kSa7)), dbl(kSa6)), s6), t);
        S = add(S, mul(mul(s4, s4), dbl(kSa8)));
    } else {  // 1/0.35 <= |x| < 6
        R = add(mul(add(mul(s, dbl(kRb3)), dbl(kRb2)), s2), add(mul(dbl(kRb1), s), dbl(kRb0)));
        R = add(R, mul(add(mul(dbl(kRb5), s), dbl(kRb4)), s4));
        R = add(R, mul(dbl(kRb6), s6));
        const double t = add(mul(s2, add(mul(dbl(kSb3), s), dbl(kSb2))), add(mul(dbl(kSb1), s), 1.0));
        S = add(mul(s4, add(mul(dbl(kSb5), s), dbl(kSb4))), t);
        S = add(S, mul(add(mul(s, dbl(kSb7)), dbl(kSb6)), s6));
    }
    const double z = dbl(bits(ax) & 0xffffffff00000000ULL);
    const double e1 = gm::exp(sub(mul(-z, z), 0.5625));
    const double e2 = gm::exp(add(mul(sub(z, ax), add(z, ax)), div(R, S)));
    const double r = mul(e2, e1);
    return neg ? sub(div(r, ax), 1.0) : sub(1.0, div(r, ax));
}

}  // namespace gm
}  // namespace ls
