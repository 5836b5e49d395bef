/*
 * zo2_rng.h -- counter-based Gaussian direction z, bit-exact with the
 * reference (shared by host C++ and sm_100a device code).
 *
 * Reference: /root/reference/pkg/src/zo2lab/numerics.py
 *   raw_uint64     :161-168  numpy Philox4x64-10 (numpy 2.3.5), key =
 *                            (stream << 64) | seed; absolute position p is
 *                            lane p % 4 of the block with 256-bit counter
 *                            p / 4 + 1 (numpy increments before generating).
 *   gaussian_fill  :171-182  u = ((r >> 11) + 0.5) * 2^-53 ; z = ndtri(u)
 *                            with scipy 1.18.1 scipy.special.ndtri (Cephes).
 *   derive_step_seed :185-190 splitmix64 finaliser.
 *
 * Bit-exactness rules (the reference computes every z in plain IEEE double):
 *  - ndtri is evaluated as separate multiply / add / divide / sqrt, never
 *    FMA-contracted (device: __dmul_rn/__dadd_rn/...; host: the library is
 *    compiled with -ffp-contract=off).
 *  - Cephes calls libm log.  On the reference's platform that is glibc 2.39
 *    x86_64 `log` (FMA ifunc variant, glibc sysdeps/ieee754/dbl-64/e_log.c),
 *    which is NOT correctly rounded (~1e-4 of inputs differ from the correctly
 *    rounded value), so zo2_log restates that exact algorithm: 128-entry
 *    (invc, logc) table, r = fma(z, invc, -1), and the same fma/add
 *    evaluation order as the compiled routine.  Constants below were read
 *    from the installed libm.so.6 (GLIBC 2.39-0ubuntu8.5, __log_data).
 *    Domain used here: normal, positive x outside [1-2^-4, 1+0x1.09p-4);
 *    ndtri only feeds it y in [2^-54, 0.1354) and sqrt(-2 log y) in (2, 8.7).
 */
#pragma once
#include <stdint.h>
#include <math.h>

#if defined(__CUDACC__)
#define ZO2_HD __host__ __device__ __forceinline__
#else
#define ZO2_HD static inline
#endif

#if defined(__CUDA_ARCH__)
#define ZO2_DMUL(a, b) __dmul_rn((a), (b))
#define ZO2_DADD(a, b) __dadd_rn((a), (b))
#define ZO2_DSUB(a, b) __dsub_rn((a), (b))
#define ZO2_DDIV(a, b) __ddiv_rn((a), (b))
#define ZO2_DSQRT(a) __dsqrt_rn((a))
#define ZO2_DFMA(a, b, c) __fma_rn((a), (b), (c))
#else
#define ZO2_DMUL(a, b) ((a) * (b))
#define ZO2_DADD(a, b) ((a) + (b))
#define ZO2_DSUB(a, b) ((a) - (b))
#define ZO2_DDIV(a, b) ((a) / (b))
#define ZO2_DSQRT(a) sqrt((a))
#define ZO2_DFMA(a, b, c) fma((a), (b), (c))
#endif

#define ZO2_LOG_CONST static const
ZO2_LOG_CONST double ZO2_LOG_LN2HI = 0x1.62e42fefa38p-1;
ZO2_LOG_CONST double ZO2_LOG_LN2LO = 0x1.ef35793c7673p-45;
ZO2_LOG_CONST double ZO2_LOG_AH[5] = {-0x1.0000000000001p-1, 0x1.555555551305bp-2, -0x1.fffffffeb459p-3, 0x1.999b324f10111p-3, -0x1.55575e506c89fp-3};
/* {invc, logc} for the 128 subintervals of [0x1.6p-1, 0x1.6p+0) */
ZO2_LOG_CONST double ZO2_LOG_TAB_H[256] = {
  0x1.734f0c3e0de9fp+0, -0x1.7cc7f79e69p-2,
  0x1.713786a2ce91fp+0, -0x1.76feec20dp-2,
  0x1.6f26008fab5ap+0, -0x1.713e31351ep-2,
  0x1.6d1a61f138c7dp+0, -0x1.6b85b382878p-2,
  0x1.6b1490bc5b4d1p+0, -0x1.65d55908078p-2,
  0x1.69147332f0cbap+0, -0x1.602d07618p-2,
  0x1.6719f18224223p+0, -0x1.5a8ca86909p-2,
  0x1.6524f99a51ed9p+0, -0x1.54f4356035p-2,
  0x1.63356aa8f24c4p+0, -0x1.4f637c36b4p-2,
  0x1.614b36b9ddc14p+0, -0x1.49da7fda85p-2,
  0x1.5f66452c65c4cp+0, -0x1.445923989a8p-2,
  0x1.5d867b5912c4fp+0, -0x1.3edf439b0b8p-2,
  0x1.5babccb5b90dep+0, -0x1.396ce448f7p-2,
  0x1.59d61f2d91a78p+0, -0x1.3401e17bdap-2,
  0x1.5805612465687p+0, -0x1.2e9e2ef468p-2,
  0x1.56397cee76bd3p+0, -0x1.2941b3830ep-2,
  0x1.54725e2a77f93p+0, -0x1.23ec58cda88p-2,
  0x1.52aff42064583p+0, -0x1.1e9e129279p-2,
  0x1.50f22dbb2bddfp+0, -0x1.1956d2b48f8p-2,
  0x1.4f38f4734ded7p+0, -0x1.141679ab9f8p-2,
  0x1.4d843cfde284p+0, -0x1.0edd094ef98p-2,
  0x1.4bd3ec078a3c8p+0, -0x1.09aa518db1p-2,
  0x1.4a27fc3e0258ap+0, -0x1.047e65263b8p-2,
  0x1.4880524d48434p+0, -0x1.feb224586fp-3,
  0x1.46dce1b192d0bp+0, -0x1.f474a7517bp-3,
  0x1.453d9d3391854p+0, -0x1.ea4443d103p-3,
  0x1.43a2744b4845ap+0, -0x1.e020d44e9bp-3,
  0x1.420b54115f8fbp+0, -0x1.d60a22977fp-3,
  0x1.40782da3ef4b1p+0, -0x1.cc00104959p-3,
  0x1.3ee8f5d57fe8fp+0, -0x1.c202956891p-3,
  0x1.3d5d9a00b4ce9p+0, -0x1.b81178d811p-3,
  0x1.3bd60c010c12bp+0, -0x1.ae2c9ccd3dp-3,
  0x1.3a5242b75dab8p+0, -0x1.a45402e129p-3,
  0x1.38d22cd9fd002p+0, -0x1.9a877681dfp-3,
  0x1.3755bc5847a1cp+0, -0x1.90c6d69483p-3,
  0x1.35dce49ad36e2p+0, -0x1.87120a645cp-3,
  0x1.34679984dd44p+0, -0x1.7d68fb4143p-3,
  0x1.32f5cceffcb24p+0, -0x1.73cb83c627p-3,
  0x1.3187775a10d49p+0, -0x1.6a39a9b376p-3,
  0x1.301c8373e399p+0, -0x1.60b3154b7ap-3,
  0x1.2eb4ebb95f841p+0, -0x1.5737d76243p-3,
  0x1.2d50a0219a9d1p+0, -0x1.4dc7b8fc23p-3,
  0x1.2bef9a8b7fd2ap+0, -0x1.4462c51d2p-3,
  0x1.2a91c7a0c1babp+0, -0x1.3b08abc83p-3,
  0x1.293726014b53p+0, -0x1.31b996b49p-3,
  0x1.27dfa5757a1f5p+0, -0x1.2875490a44p-3,
  0x1.268b39b1d3bbfp+0, -0x1.1f3b9f879ap-3,
  0x1.2539d838ff5bdp+0, -0x1.160c8252cap-3,
  0x1.23eb7aac9083bp+0, -0x1.0ce7f57f72p-3,
  0x1.22a012ba940b6p+0, -0x1.03cdc49feap-3,
  0x1.2157996cc4132p+0, -0x1.f57bdbc4b8p-4,
  0x1.201201dd2fc9bp+0, -0x1.e370896404p-4,
  0x1.1ecf4494d480bp+0, -0x1.d17983ef94p-4,
  0x1.1d8f5528f6569p+0, -0x1.bf9674ed8ap-4,
  0x1.1c52311577e7cp+0, -0x1.adc79202f6p-4,
  0x1.1b17c74cb26e9p+0, -0x1.9c0c3e7288p-4,
  0x1.19e010c2c1ab6p+0, -0x1.8a646b372cp-4,
  0x1.18ab07bb670bdp+0, -0x1.78d01b3acp-4,
  0x1.1778a25efbcb6p+0, -0x1.674f14538p-4,
  0x1.1648d354c31dap+0, -0x1.55e0e6d878p-4,
  0x1.151b990275fddp+0, -0x1.4485cdea1ep-4,
  0x1.13f0ea432d24cp+0, -0x1.333d94d6aap-4,
  0x1.12c8b7210f9dap+0, -0x1.22079f8c56p-4,
  0x1.11a3028ecb531p+0, -0x1.10e4698622p-4,
  0x1.107fbda8434afp+0, -0x1.ffa6c6ad2p-5,
  0x1.0f5ee0f4e6bb3p+0, -0x1.dda8d4a774p-5,
  0x1.0e4065d2a9fcep+0, -0x1.bbcece485p-5,
  0x1.0d244632ca521p+0, -0x1.9a1894012cp-5,
  0x1.0c0a77ce2981ap+0, -0x1.788583302cp-5,
  0x1.0af2f83c636d1p+0, -0x1.5715e67d68p-5,
  0x1.09ddb98a01339p+0, -0x1.35c8a49658p-5,
  0x1.08cabaf52e7dfp+0, -0x1.149e364154p-5,
  0x1.07b9f2f4e28fbp+0, -0x1.e72c082eb8p-6,
  0x1.06ab58c358f19p+0, -0x1.a55f152528p-6,
  0x1.059eea5ecf92cp+0, -0x1.63d62cf818p-6,
  0x1.04949cdd12c9p+0, -0x1.228fb8caap-6,
  0x1.038c6c6f0ada9p+0, -0x1.c317b20f9p-7,
  0x1.02865137932a9p+0, -0x1.419355daap-7,
  0x1.0182427ea7348p+0, -0x1.81203c2ecp-8,
  0x1.008040614b195p+0, -0x1.004097924p-9,
  0x1.fe01ff726fa1ap-1, 0x1.feff3849p-9,
  0x1.fa11cc261ea74p-1, 0x1.7dc41353dp-7,
  0x1.f6310b081992ep-1, 0x1.3cea3c4c28p-6,
  0x1.f25f63ceeadcdp-1, 0x1.b9fc11489p-6,
  0x1.ee9c8039113e7p-1, 0x1.1b0d8ce11p-5,
  0x1.eae8078cbb1abp-1, 0x1.58a5bd001cp-5,
  0x1.e741aa29d0c9bp-1, 0x1.95c8340d88p-5,
  0x1.e3a91830a99b5p-1, 0x1.d276aef578p-5,
  0x1.e01e009609a56p-1, 0x1.07598e598cp-4,
  0x1.dca01e577bb98p-1, 0x1.253f5e30d2p-4,
  0x1.d92f20b7c9103p-1, 0x1.42edd8b38p-4,
  0x1.d5cac66fb5ccep-1, 0x1.606598757cp-4,
  0x1.d272caa5ede9dp-1, 0x1.7da76356ap-4,
  0x1.cf26e3e6b2ccdp-1, 0x1.9ab434e1c6p-4,
  0x1.cbe6da2a77902p-1, 0x1.b78c7bb0d6p-4,
  0x1.c8b266d37086dp-1, 0x1.d431332e72p-4,
  0x1.c5894bd5d5804p-1, 0x1.f0a3171de6p-4,
  0x1.c26b533bb9f8cp-1, 0x1.067152b914p-3,
  0x1.bf583eeece73fp-1, 0x1.147858292bp-3,
  0x1.bc4fd75db96c1p-1, 0x1.2266ecdca3p-3,
  0x1.b951e0c864a28p-1, 0x1.303d7a6c55p-3,
  0x1.b65e2c5ef3e2cp-1, 0x1.3dfc33c331p-3,
  0x1.b374867c9888bp-1, 0x1.4ba366b7a8p-3,
  0x1.b094b211d304ap-1, 0x1.5933928d1fp-3,
  0x1.adbe885f2ef7ep-1, 0x1.66acd2418fp-3,
  0x1.aaf1d31603da2p-1, 0x1.740f8ec669p-3,
  0x1.a82e63fd358a7p-1, 0x1.815c0f51afp-3,
  0x1.a5740ef09738bp-1, 0x1.8e92954f68p-3,
  0x1.a2c2a90ab4b27p-1, 0x1.9bb3602f84p-3,
  0x1.a01a01393f2d1p-1, 0x1.a8bed1c2cp-3,
  0x1.9d79f24db3c1bp-1, 0x1.b5b515c01dp-3,
  0x1.9ae2505c7b19p-1, 0x1.c2967ccbccp-3,
  0x1.9852ef297ce2fp-1, 0x1.cf635d5486p-3,
  0x1.95cbaeea44b75p-1, 0x1.dc1bd3446cp-3,
  0x1.934c69de74838p-1, 0x1.e8c01b8cfep-3,
  0x1.90d4f2f6752e6p-1, 0x1.f5509c0179p-3,
  0x1.8e6528effd79dp-1, 0x1.00e6c121fb8p-2,
  0x1.8bfce9fcc007cp-1, 0x1.071b80e93dp-2,
  0x1.899c0dabec30ep-1, 0x1.0d46b9e867p-2,
  0x1.87427aa2317fbp-1, 0x1.13687334bdp-2,
  0x1.84f00acb39a08p-1, 0x1.1980d672348p-2,
  0x1.82a49e8653e55p-1, 0x1.1f8ffe0cc8p-2,
  0x1.8060195f4026p-1, 0x1.2595fd76368p-2,
  0x1.7e22563e0a329p-1, 0x1.2b9300914a8p-2,
  0x1.7beb377dcb5adp-1, 0x1.3187210436p-2,
  0x1.79baa679725c2p-1, 0x1.377266dec18p-2,
  0x1.77907f2170657p-1, 0x1.3d54ffbaf3p-2,
  0x1.756cadbd6130cp-1, 0x1.432eee32fep-2,
};

#if defined(__CUDACC__)
static __constant__ double ZO2_LOG_AD[5] = {-0x1.0000000000001p-1, 0x1.555555551305bp-2, -0x1.fffffffeb459p-3, 0x1.999b324f10111p-3, -0x1.55575e506c89fp-3};
#endif
#if defined(__CUDA_ARCH__)
#define ZO2_LOG_A ZO2_LOG_AD
#else
#define ZO2_LOG_A ZO2_LOG_AH
#endif
#if defined(__CUDACC__)
/* device copy of the table (global memory: per-lane indices diverge, so
 * constant memory would serialise) */
static __device__ const double ZO2_LOG_TAB_D[256] = {
  0x1.734f0c3e0de9fp+0, -0x1.7cc7f79e69p-2,
  0x1.713786a2ce91fp+0, -0x1.76feec20dp-2,
  0x1.6f26008fab5ap+0, -0x1.713e31351ep-2,
  0x1.6d1a61f138c7dp+0, -0x1.6b85b382878p-2,
  0x1.6b1490bc5b4d1p+0, -0x1.65d55908078p-2,
  0x1.69147332f0cbap+0, -0x1.602d07618p-2,
  0x1.6719f18224223p+0, -0x1.5a8ca86909p-2,
  0x1.6524f99a51ed9p+0, -0x1.54f4356035p-2,
  0x1.63356aa8f24c4p+0, -0x1.4f637c36b4p-2,
  0x1.614b36b9ddc14p+0, -0x1.49da7fda85p-2,
  0x1.5f66452c65c4cp+0, -0x1.445923989a8p-2,
  0x1.5d867b5912c4fp+0, -0x1.3edf439b0b8p-2,
  0x1.5babccb5b90dep+0, -0x1.396ce448f7p-2,
  0x1.59d61f2d91a78p+0, -0x1.3401e17bdap-2,
  0x1.5805612465687p+0, -0x1.2e9e2ef468p-2,
  0x1.56397cee76bd3p+0, -0x1.2941b3830ep-2,
  0x1.54725e2a77f93p+0, -0x1.23ec58cda88p-2,
  0x1.52aff42064583p+0, -0x1.1e9e129279p-2,
  0x1.50f22dbb2bddfp+0, -0x1.1956d2b48f8p-2,
  0x1.4f38f4734ded7p+0, -0x1.141679ab9f8p-2,
  0x1.4d843cfde284p+0, -0x1.0edd094ef98p-2,
  0x1.4bd3ec078a3c8p+0, -0x1.09aa518db1p-2,
  0x1.4a27fc3e0258ap+0, -0x1.047e65263b8p-2,
  0x1.4880524d48434p+0, -0x1.feb224586fp-3,
  0x1.46dce1b192d0bp+0, -0x1.f474a7517bp-3,
  0x1.453d9d3391854p+0, -0x1.ea4443d103p-3,
  0x1.43a2744b4845ap+0, -0x1.e020d44e9bp-3,
  0x1.420b54115f8fbp+0, -0x1.d60a22977fp-3,
  0x1.40782da3ef4b1p+0, -0x1.cc00104959p-3,
  0x1.3ee8f5d57fe8fp+0, -0x1.c202956891p-3,
  0x1.3d5d9a00b4ce9p+0, -0x1.b81178d811p-3,
  0x1.3bd60c010c12bp+0, -0x1.ae2c9ccd3dp-3,
  0x1.3a5242b75dab8p+0, -0x1.a45402e129p-3,
  0x1.38d22cd9fd002p+0, -0x1.9a877681dfp-3,
  0x1.3755bc5847a1cp+0, -0x1.90c6d69483p-3,
  0x1.35dce49ad36e2p+0, -0x1.87120a645cp-3,
  0x1.34679984dd44p+0, -0x1.7d68fb4143p-3,
  0x1.32f5cceffcb24p+0, -0x1.73cb83c627p-3,
  0x1.3187775a10d49p+0, -0x1.6a39a9b376p-3,
  0x1.301c8373e399p+0, -0x1.60b3154b7ap-3,
  0x1.2eb4ebb95f841p+0, -0x1.5737d76243p-3,
  0x1.2d50a0219a9d1p+0, -0x1.4dc7b8fc23p-3,
  0x1.2bef9a8b7fd2ap+0, -0x1.4462c51d2p-3,
  0x1.2a91c7a0c1babp+0, -0x1.3b08abc83p-3,
  0x1.293726014b53p+0, -0x1.31b996b49p-3,
  0x1.27dfa5757a1f5p+0, -0x1.2875490a44p-3,
  0x1.268b39b1d3bbfp+0, -0x1.1f3b9f879ap-3,
  0x1.2539d838ff5bdp+0, -0x1.160c8252cap-3,
  0x1.23eb7aac9083bp+0, -0x1.0ce7f57f72p-3,
  0x1.22a012ba940b6p+0, -0x1.03cdc49feap-3,
  0x1.2157996cc4132p+0, -0x1.f57bdbc4b8p-4,
  0x1.201201dd2fc9bp+0, -0x1.e370896404p-4,
  0x1.1ecf4494d480bp+0, -0x1.d17983ef94p-4,
  0x1.1d8f5528f6569p+0, -0x1.bf9674ed8ap-4,
  0x1.1c52311577e7cp+0, -0x1.adc79202f6p-4,
  0x1.1b17c74cb26e9p+0, -0x1.9c0c3e7288p-4,
  0x1.19e010c2c1ab6p+0, -0x1.8a646b372cp-4,
  0x1.18ab07bb670bdp+0, -0x1.78d01b3acp-4,
  0x1.1778a25efbcb6p+0, -0x1.674f14538p-4,
  0x1.1648d354c31dap+0, -0x1.55e0e6d878p-4,
  0x1.151b990275fddp+0, -0x1.4485cdea1ep-4,
  0x1.13f0ea432d24cp+0, -0x1.333d94d6aap-4,
  0x1.12c8b7210f9dap+0, -0x1.22079f8c56p-4,
  0x1.11a3028ecb531p+0, -0x1.10e4698622p-4,
  0x1.107fbda8434afp+0, -0x1.ffa6c6ad2p-5,
  0x1.0f5ee0f4e6bb3p+0, -0x1.dda8d4a774p-5,
  0x1.0e4065d2a9fcep+0, -0x1.bbcece485p-5,
  0x1.0d244632ca521p+0, -0x1.9a1894012cp-5,
  0x1.0c0a77ce2981ap+0, -0x1.788583302cp-5,
  0x1.0af2f83c636d1p+0, -0x1.5715e67d68p-5,
  0x1.09ddb98a01339p+0, -0x1.35c8a49658p-5,
  0x1.08cabaf52e7dfp+0, -0x1.149e364154p-5,
  0x1.07b9f2f4e28fbp+0, -0x1.e72c082eb8p-6,
  0x1.06ab58c358f19p+0, -0x1.a55f152528p-6,
  0x1.059eea5ecf92cp+0, -0x1.63d62cf818p-6,
  0x1.04949cdd12c9p+0, -0x1.228fb8caap-6,
  0x1.038c6c6f0ada9p+0, -0x1.c317b20f9p-7,
  0x1.02865137932a9p+0, -0x1.419355daap-7,
  0x1.0182427ea7348p+0, -0x1.81203c2ecp-8,
  0x1.008040614b195p+0, -0x1.004097924p-9,
  0x1.fe01ff726fa1ap-1, 0x1.feff3849p-9,
  0x1.fa11cc261ea74p-1, 0x1.7dc41353dp-7,
  0x1.f6310b081992ep-1, 0x1.3cea3c4c28p-6,
  0x1.f25f63ceeadcdp-1, 0x1.b9fc11489p-6,
  0x1.ee9c8039113e7p-1, 0x1.1b0d8ce11p-5,
  0x1.eae8078cbb1abp-1, 0x1.58a5bd001cp-5,
  0x1.e741aa29d0c9bp-1, 0x1.95c8340d88p-5,
  0x1.e3a91830a99b5p-1, 0x1.d276aef578p-5,
  0x1.e01e009609a56p-1, 0x1.07598e598cp-4,
  0x1.dca01e577bb98p-1, 0x1.253f5e30d2p-4,
  0x1.d92f20b7c9103p-1, 0x1.42edd8b38p-4,
  0x1.d5cac66fb5ccep-1, 0x1.606598757cp-4,
  0x1.d272caa5ede9dp-1, 0x1.7da76356ap-4,
  0x1.cf26e3e6b2ccdp-1, 0x1.9ab434e1c6p-4,
  0x1.cbe6da2a77902p-1, 0x1.b78c7bb0d6p-4,
  0x1.c8b266d37086dp-1, 0x1.d431332e72p-4,
  0x1.c5894bd5d5804p-1, 0x1.f0a3171de6p-4,
  0x1.c26b533bb9f8cp-1, 0x1.067152b914p-3,
  0x1.bf583eeece73fp-1, 0x1.147858292bp-3,
  0x1.bc4fd75db96c1p-1, 0x1.2266ecdca3p-3,
  0x1.b951e0c864a28p-1, 0x1.303d7a6c55p-3,
  0x1.b65e2c5ef3e2cp-1, 0x1.3dfc33c331p-3,
  0x1.b374867c9888bp-1, 0x1.4ba366b7a8p-3,
  0x1.b094b211d304ap-1, 0x1.5933928d1fp-3,
  0x1.adbe885f2ef7ep-1, 0x1.66acd2418fp-3,
  0x1.aaf1d31603da2p-1, 0x1.740f8ec669p-3,
  0x1.a82e63fd358a7p-1, 0x1.815c0f51afp-3,
  0x1.a5740ef09738bp-1, 0x1.8e92954f68p-3,
  0x1.a2c2a90ab4b27p-1, 0x1.9bb3602f84p-3,
  0x1.a01a01393f2d1p-1, 0x1.a8bed1c2cp-3,
  0x1.9d79f24db3c1bp-1, 0x1.b5b515c01dp-3,
  0x1.9ae2505c7b19p-1, 0x1.c2967ccbccp-3,
  0x1.9852ef297ce2fp-1, 0x1.cf635d5486p-3,
  0x1.95cbaeea44b75p-1, 0x1.dc1bd3446cp-3,
  0x1.934c69de74838p-1, 0x1.e8c01b8cfep-3,
  0x1.90d4f2f6752e6p-1, 0x1.f5509c0179p-3,
  0x1.8e6528effd79dp-1, 0x1.00e6c121fb8p-2,
  0x1.8bfce9fcc007cp-1, 0x1.071b80e93dp-2,
  0x1.899c0dabec30ep-1, 0x1.0d46b9e867p-2,
  0x1.87427aa2317fbp-1, 0x1.13687334bdp-2,
  0x1.84f00acb39a08p-1, 0x1.1980d672348p-2,
  0x1.82a49e8653e55p-1, 0x1.1f8ffe0cc8p-2,
  0x1.8060195f4026p-1, 0x1.2595fd76368p-2,
  0x1.7e22563e0a329p-1, 0x1.2b9300914a8p-2,
  0x1.7beb377dcb5adp-1, 0x1.3187210436p-2,
  0x1.79baa679725c2p-1, 0x1.377266dec18p-2,
  0x1.77907f2170657p-1, 0x1.3d54ffbaf3p-2,
  0x1.756cadbd6130cp-1, 0x1.432eee32fep-2,
};

#endif

ZO2_HD uint64_t zo2_as_u64(double x) {
#if defined(__CUDA_ARCH__)
  return (uint64_t)__double_as_longlong(x);
#else
  union { double d; uint64_t u; } c; c.d = x; return c.u;
#endif
}
ZO2_HD double zo2_as_f64(uint64_t u) {
#if defined(__CUDA_ARCH__)
  return __longlong_as_double((long long)u);
#else
  union { double d; uint64_t u; } c; c.u = u; return c.d;
#endif
}

/* glibc 2.39 log, main path (see header comment for the domain). */
ZO2_HD double zo2_log(double x) {
#if defined(__CUDA_ARCH__)
  const double *tab = ZO2_LOG_TAB_D;
#else
  const double *tab = ZO2_LOG_TAB_H;
#endif
  const uint64_t ix = zo2_as_u64(x);
  const uint64_t tmp = ix - 0x3fe6000000000000ULL;
  const int i = (int)((tmp >> 45) & 127);
  const int k = (int)((int64_t)tmp >> 52);
  const uint64_t iz = ix - (tmp & (0xfffULL << 52));
  const double invc = tab[2 * i], logc = tab[2 * i + 1];
  const double z = zo2_as_f64(iz);
  const double kd = (double)k;
  const double w = ZO2_DFMA(kd, ZO2_LOG_LN2HI, logc);
  const double r = ZO2_DFMA(z, invc, -1.0);
  const double t1 = ZO2_DFMA(r, ZO2_LOG_A[2], ZO2_LOG_A[1]);
  const double hi = ZO2_DADD(r, w);
  const double r2 = ZO2_DMUL(r, r);
  double lo = ZO2_DADD(ZO2_DSUB(w, hi), r);
  lo = ZO2_DFMA(kd, ZO2_LOG_LN2LO, lo);
  const double r3 = ZO2_DMUL(r, r2);
  const double t2 = ZO2_DFMA(r, ZO2_LOG_A[4], ZO2_LOG_A[3]);
  const double u = ZO2_DFMA(r2, ZO2_LOG_A[0], lo);
  const double p = ZO2_DFMA(t2, r2, t1);
  const double v = ZO2_DFMA(r3, p, u);
  return ZO2_DADD(v, hi);
}

/* ------------------------------------------------------------ Philox4x64 */
#ifndef ZO2_MULHILO_EXPLICIT
#define ZO2_MULHILO_EXPLICIT 0
#endif
ZO2_HD void zo2_mulhilo64(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
#if defined(__CUDA_ARCH__) && !ZO2_MULHILO_EXPLICIT
  *lo = a * b;
  *hi = __umul64hi(a, b);
#elif defined(__CUDA_ARCH__)
  // 128-bit product from four 32x32->64 multiply-adds (IMAD.WIDE.U32), the
  // partial products shared between the high and the low half
  const uint32_t al = (uint32_t)a, ah = (uint32_t)(a >> 32);
  const uint32_t bl = (uint32_t)b, bh = (uint32_t)(b >> 32);
  const uint64_t p0 = (uint64_t)al * bl;
  const uint64_t t = (uint64_t)al * bh + (p0 >> 32);
  const uint64_t u = (uint64_t)ah * bl + (uint32_t)t;
  *lo = (u << 32) | (uint32_t)p0;
  *hi = (uint64_t)ah * bh + (t >> 32) + (u >> 32);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (uint64_t)p;
  *hi = (uint64_t)(p >> 64);
#endif
}

/* One Philox4x64-10 block for 256-bit counter (c0, c1, 0, 0). */
ZO2_HD void zo2_philox4x64(uint64_t c0, uint64_t c1, uint64_t k0, uint64_t k1,
                           uint64_t out[4]) {
  uint64_t x0 = c0, x1 = c1, x2 = 0, x3 = 0;
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, lo0, hi1, lo1;
    zo2_mulhilo64(0xD2E7470EE14C6C93ULL, x0, &hi0, &lo0);
    zo2_mulhilo64(0xCA5A826395121157ULL, x2, &hi1, &lo1);
    const uint64_t n0 = hi1 ^ x1 ^ k0;
    const uint64_t n2 = hi0 ^ x3 ^ k1;
    x0 = n0; x1 = lo1; x2 = n2; x3 = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  out[0] = x0; out[1] = x1; out[2] = x2; out[3] = x3;
}

/* The four raw draws of block b = p / 4 (positions 4b .. 4b+3). */
ZO2_HD void zo2_raw_block(uint64_t seed, uint64_t stream, uint64_t b,
                          uint64_t out[4]) {
  const uint64_t c0 = b + 1;
  zo2_philox4x64(c0, c0 == 0 ? 1ULL : 0ULL, seed, stream, out);
}

/* ------------------------------------------------------- Cephes ndtri */
ZO2_HD double zo2_polevl(double x, const double *c, int n) {
  double a = c[0];
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int i = 1; i <= n; ++i) a = ZO2_DADD(ZO2_DMUL(a, x), c[i]);
  return a;
}
ZO2_HD double zo2_p1evl(double x, const double *c, int n) {
  double a = ZO2_DADD(x, c[0]);
#if defined(__CUDA_ARCH__)
#pragma unroll
#endif
  for (int i = 1; i < n; ++i) a = ZO2_DADD(ZO2_DMUL(a, x), c[i]);
  return a;
}

#define ZO2_NDTRI_P0 {-5.99633501014107895267E1, 9.80010754185999661536E1, -5.66762857469070293439E1, 1.39312609387279679503E1, -1.23916583867381258016E0}
#define ZO2_NDTRI_Q0 {1.95448858338141759834E0, 4.67627912898881538453E0, 8.63602421390890590575E1, -2.25462687854119370527E2, 2.00260212380060660359E2, -8.20372256168333339912E1, 1.59056225126211695515E1, -1.18331621121330003142E0}
#define ZO2_NDTRI_P1 {4.05544892305962419923E0, 3.15251094599893866154E1, 5.71628192246421288162E1, 4.40805073893200834700E1, 1.46849561928858024014E1, 2.18663306850790267539E0, -1.40256079171354495875E-1, -3.50424626827848203418E-2, -8.57456785154685413611E-4}
#define ZO2_NDTRI_Q1 {1.57799883256466749731E1, 4.53907635128879210584E1, 4.13172038254672030440E1, 1.50425385692907503408E1, 2.50464946208309415979E0, -1.42182922854787788574E-1, -3.80806407691578277194E-2, -9.33259480895457427372E-4}
#define ZO2_NDTRI_P2 {3.23774891776946035970E0, 6.91522889068984211695E0, 3.93881025292474443415E0, 1.33303460815807542389E0, 2.01485389549179081538E-1, 1.23716634817820021358E-2, 3.01581553508235416007E-4, 2.65806974686737550832E-6, 6.23974539184983293730E-9}
#define ZO2_NDTRI_Q2 {6.02427039364742014255E0, 3.67983563856160859403E0, 1.37702099489081330271E0, 2.16236993594496635890E-1, 1.34204006088543189037E-2, 3.28014464682127739104E-4, 2.89247864745380683936E-6, 6.79019408009981274425E-9}


/* Coefficient tables: __constant__ on the device so FP64 instructions take
 * them as c[bank][offset] operands; static arrays on the host. */
#if defined(__CUDACC__)
static __constant__ double ZO2_D_P0[5] = ZO2_NDTRI_P0;
static __constant__ double ZO2_D_Q0[8] = ZO2_NDTRI_Q0;
static __constant__ double ZO2_D_P1[9] = ZO2_NDTRI_P1;
static __constant__ double ZO2_D_Q1[8] = ZO2_NDTRI_Q1;
static __constant__ double ZO2_D_P2[9] = ZO2_NDTRI_P2;
static __constant__ double ZO2_D_Q2[8] = ZO2_NDTRI_Q2;
#endif
static const double ZO2_H_P0[5] = ZO2_NDTRI_P0;
static const double ZO2_H_Q0[8] = ZO2_NDTRI_Q0;
static const double ZO2_H_P1[9] = ZO2_NDTRI_P1;
static const double ZO2_H_Q1[8] = ZO2_NDTRI_Q1;
static const double ZO2_H_P2[9] = ZO2_NDTRI_P2;
static const double ZO2_H_Q2[8] = ZO2_NDTRI_Q2;
#ifndef ZO2_CONST_COEF
#define ZO2_CONST_COEF 1
#endif
#if defined(__CUDA_ARCH__) && ZO2_CONST_COEF
#define ZO2_DECL_COEF(var, name, n) const double *var = ZO2_D_##name;
#elif defined(__CUDA_ARCH__)
#define ZO2_DECL_COEF(var, name, n) const double var[n] = ZO2_NDTRI_##name;
#else
#define ZO2_DECL_COEF(var, name, n) const double *var = ZO2_H_##name;
#endif

/* Central branch: |y - 0.5| < 0.5 - exp(-2). */
ZO2_HD double zo2_ndtri_central(double y) {
  ZO2_DECL_COEF(P0, P0, 5)
  ZO2_DECL_COEF(Q0, Q0, 8)
  y = ZO2_DSUB(y, 0.5);
  const double y2 = ZO2_DMUL(y, y);
  const double t = ZO2_DDIV(ZO2_DMUL(y2, zo2_polevl(y2, P0, 4)), zo2_p1evl(y2, Q0, 8));
  const double x = ZO2_DADD(y, ZO2_DMUL(y, t));
  return ZO2_DMUL(x, 2.50662827463100050242E0);
}

/* Tail branch: y <= exp(-2) after reflection; code=1 negates. */
ZO2_HD double zo2_ndtri_tail(double y, int negate) {
  ZO2_DECL_COEF(P1, P1, 9)
  ZO2_DECL_COEF(Q1, Q1, 8)
  ZO2_DECL_COEF(P2, P2, 9)
  ZO2_DECL_COEF(Q2, Q2, 8)
  double x = ZO2_DSQRT(ZO2_DMUL(-2.0, zo2_log(y)));
  const double x0 = ZO2_DSUB(x, ZO2_DDIV(zo2_log(x), x));
  const double z = ZO2_DDIV(1.0, x);
  double x1;
  if (x < 8.0)
    x1 = ZO2_DDIV(ZO2_DMUL(z, zo2_polevl(z, P1, 8)), zo2_p1evl(z, Q1, 8));
  else
    x1 = ZO2_DDIV(ZO2_DMUL(z, zo2_polevl(z, P2, 8)), zo2_p1evl(z, Q2, 8));
  x = ZO2_DSUB(x0, x1);
  return negate ? -x : x;
}

/* u in (0, 1] as produced by zo2_u53 (never 0; 1.0 with probability 2^-53). */
ZO2_HD double zo2_ndtri(double y0) {
  if (y0 == 1.0) return INFINITY;
  if (y0 == 0.0) return -INFINITY;
  const double expm2 = 0.13533528323661269189;
  double y = y0;
  int negate = 1;
  if (y > ZO2_DSUB(1.0, expm2)) {
    y = ZO2_DSUB(1.0, y);
    negate = 0;
  }
  if (y > expm2) return zo2_ndtri_central(y);
  return zo2_ndtri_tail(y, negate);
}

ZO2_HD double zo2_u53(uint64_t r) {
  return ZO2_DMUL(ZO2_DADD((double)(r >> 11), 0.5), 0x1p-53);
}

ZO2_HD double zo2_gauss_at(uint64_t seed, uint64_t stream, uint64_t pos) {
  uint64_t b[4];
  zo2_raw_block(seed, stream, pos >> 2, b);
  return zo2_ndtri(zo2_u53(b[pos & 3]));
}

ZO2_HD uint64_t zo2_derive_step_seed(uint64_t base, uint64_t j) {
  uint64_t x = base ^ (j * 0x9E3779B97F4A7C15ULL);
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
