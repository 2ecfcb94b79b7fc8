// capi.cu -- the C ABI (include/pipedp_cuda.h): validation with the
// reference's rules, value-width / stage planning, device memory, launches.
//
// There is no CPU compute path in this file: every table is produced by a
// kernel from sdp_kernels.cuh / mcm_kernels.cuh, and a missing or unusable GPU
// is reported as PIPEDP_ERR_NO_DEVICE.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <random>
#include <string>
#include <thread>
#include <unordered_set>
#include <vector>

#include "../../include/pipedp_cuda.h"
#include "mcm_kernels.cuh"
#include "mcm_tiled.cuh"
#include "sdp_kernels.cuh"
#include "sdp_jump.cuh"
#include "sdp_chunked.cuh"
#include "sdp_v2.cuh"
#include "host_io.hpp"
#include "sdp_rank.hpp"
#include "sdp_batch_dom.hpp"
#include "mcm_tournament.hpp"
#include "sdp_cluster.hpp"
#include "mcm_batch.hpp"

using namespace pipedp_dev;

#include "capi_util.hpp"

using namespace pipedp_capi;

namespace {

int ceil_log2(uint64_t v) {
  int r = 0;
  while ((1ull << r) < v) ++r;
  return r;
}

// ================================================================== S-DP ===
struct SdpDispatch {
  int op;
  int bits;   // 32 or 64
  bool assoc; // regrouping legal
  bool small; // CTA: a1 < 64, warp: a1 < 32
  bool gfar;
  bool remote;  // multi-CTA: producer CTAs on other SMs
  bool warp_kernel;
  SdpShape shape;
  int threads;
  int grid_extra;  // producer CTAs (remote)
  size_t smem;
  int wpb;  // warp kernel: warps per block
  bool v2;   // offset-partitioned single-instance pipeline (sdp_v2.cuh)
  bool serial;  // tiny offset sets: one-thread chain (sdp_serial_thread)
  bool jump;    // a_1 <= 8: jump-ahead segments (sdp_jump)
  bool chunked; // one large min/max instance as a batch of chunks (sdp_chunked.cuh)
  int64_t chunk_len;  // chunk length L (a multiple of 32 with few set bits: square-and-multiply)
  int method;   // 0 pipeline, 1 the paper's tournament (prefix), 2 the paper's naive method
  SdpV2Shape s2;
  bool cluster = false;  // one instance over a thread-block cluster (sdp_cluster.cu)
  bool vals32 = false;   // the paper's methods: every value of the instance fits int32 (a 4-byte ring)
  pipedp_cluster::ClusterPlan cplan{};
};

// value width and associativity from the init values (see common.cuh)
void sdp_value_class(int op, const int64_t* init, int64_t count, int* bits, bool* assoc) {
  bool fits32 = true, any_pos = false, any_neg = false;
  for (int64_t i = 0; i < count; ++i) {
    const int64_t v = init[i];
    if (op == PIPEDP_OP_MODULAR_ADD) fits32 = fits32 && v >= 0 && v < kModulus;
    else fits32 = fits32 && v >= INT32_MIN && v <= INT32_MAX;
    any_pos = any_pos || v > 0;
    any_neg = any_neg || v < 0;
  }
  *bits = (op != PIPEDP_OP_SATURATING_ADD && fits32) ? 32 : 64;
  *assoc = op != PIPEDP_OP_SATURATING_ADD || !(any_pos && any_neg);
}

constexpr size_t kSmemBudget = 200 * 1024;
constexpr int kAMid = 256;
constexpr int kARemote = 1024;

// Dispatch switches: each one selects or disables an
// alternative kernel path so the tests can reach it; the defaults are the
// product.  Any other PIPEDP_* name is a tuning constant -- the environment is
// not consulted for it.
int env_int(const char* name, int dflt) {
  static const char* const kSwitches[] = {
      "PIPEDP_SDP_CHUNKED", "PIPEDP_SDP_RANK",     "PIPEDP_SDP_BDOM",      "PIPEDP_SDP_CLUSTER",
      "PIPEDP_SDP_V2",      "PIPEDP_SDP_MULTI",    "PIPEDP_SDP_JUMP",      "PIPEDP_SDP_SERIAL",
      "PIPEDP_SDP_REMOTE_WARPS", "PIPEDP_SDP_REMOTE_CTAS", "PIPEDP_SDP_MID_WARPS", "PIPEDP_SDP_AREMOTE",
      "PIPEDP_SDP2_WRITERS", "PIPEDP_CHUNK_OVERLAP", "PIPEDP_MCM_TILED",   "PIPEDP_MCM_T32_MAXN",
      "PIPEDP_MCM_BLOCKED", "PIPEDP_MCM_SQUARE",   "PIPEDP_MCM_BATCH_WARP", "PIPEDP_MCM_PACKED_SQUARE",
      "PIPEDP_D2H_NARROW",  "PIPEDP_STREAM_D2H",   "PIPEDP_D2H_PROGRESSIVE"};
  bool known = false;
  for (const char* k : kSwitches) known = known || strcmp(k, name) == 0;
  if (!known) return dflt;
  const char* v = getenv(name);
  return v && *v ? atoi(v) : dflt;
}

int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) != cudaSuccess || cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess) {
    (void)cudaGetLastError();
    return 148;
  }
  return sms;
}

size_t sdp_cta_smem(int64_t R, int64_t kpad, size_t vb) {
  return 2 * R * vb + 3 * kpad * 4 + (size_t)(kMidSlots + kFarSlots) * 32 * vb +
         (size_t)(2 * kBatchBars + kMidSlots + kFarSlots) * 8 + 64;
}

size_t sdp_v2_smem(int64_t R, int64_t kpad, size_t vb, int NW, int NC) {
  return 2 * R * vb + kpad * 4 + (size_t)kMidSlots * 32 * vb + (size_t)kNearSlots * NW * 32 * vb +
         (size_t)kFetchSlots * 32 * vb + (size_t)kPreMax * 32 * 4 + 16 +
         (size_t)(2 * kBatchBars + kMidSlots + kNearSlots + kFetchSlots) * 8 + 64;
}

// sdp_v2 plan (one instance): offsets >= a_rem to remote producers (when there
// are enough of them), [64, a_rem) to register-resident near warps, < 64 to the
// chain / combiners.  Returns false when the instance does not fit the layout.
bool plan_sdp_v2(int64_t n, int64_t k, int64_t a1, const int64_t* offs, SdpDispatch* d) {
  const size_t vb = d->bits / 8;
  SdpV2Shape& s = d->s2;
  s.n = n;
  s.k = (int32_t)k;
  s.a1 = (int32_t)a1;
  const int64_t kpad = (k + 3) & ~3ll;
  const int64_t nb = (n - a1 + 31) / 32;
  int a_rem = std::max(128, env_int("PIPEDP_SDP2_AREM", 768));
  // chain-local range [l+33, a_chain): at most kPreMax offsets for lane 0
  // chain-local range: [l+33, 64) per lane (<= 31 offsets) plus the
  // lane-independent [64, a_chain) with at most kPreUMax offsets
  int a_chain = 64;
  for (int cand = 96; cand <= 256; cand += 32) {
    int64_t cnt = 0;
    for (int64_t j = 0; j < k; ++j) cnt += offs[j] >= 64 && offs[j] < cand;
    if (cnt <= kPreUMax) a_chain = cand;
  }
  a_chain = std::min(a_chain, std::max(64, env_int("PIPEDP_SDP2_ACHAIN", 1 << 20)));
  // dominance form (sdp_v2.cuh): min/max with offset 1 take [l+33, 128) from
  // the chain's own shuffles once batch 3 is reached (the first batches fold
  // the same range from the ring, so [64, 128) must fit the register list)
  bool has1 = false;
  int64_t n64_128 = 0;
  for (int64_t j = 0; j < k; ++j) {
    has1 = has1 || offs[j] == 1;
    n64_128 += offs[j] >= 64 && offs[j] < 128;
  }
  // the dominance form takes [l+33, a_chain) with one shuffle per 32-wide
  // range (a_chain up to 256: near warps then see >= 8 batches of look-ahead);
  // its first a_chain/32 - 1 batches fold that range from the ring directly
  bool dom = false;
  if ((d->op == PIPEDP_OP_MIN || d->op == PIPEDP_OP_MAX) && has1 && env_int("PIPEDP_SDP2_DOM", 1) != 0) {
    dom = true;
    a_chain = std::min(256, std::max(128, env_int("PIPEDP_SDP2_DOM_ACHAIN", 256))) & ~31;
  }
  (void)n64_128;
  int64_t jr = 0, jn = 0;
  for (int64_t j = 0; j < k; ++j) {
    jr += offs[j] >= a_rem;
    jn += offs[j] >= a_chain;
  }
  bool remote = jr >= 64 && nb >= 256 && env_int("PIPEDP_SDP_MULTI", 1) != 0;
  if (!remote) {
    a_rem = 1 << 30;
    jr = 0;
  }
  const int64_t cover = remote ? a_rem : a1;
  const int64_t R = 1ll << ceil_log2((uint64_t)(cover + 512));
  const int64_t count = jn - jr;
  const int NW = (int)((count + kNearMax - 1) / kNearMax);
  if (NW > kNearWarps) return false;
  // roles: as many combiners / near groups / fetchers as the 24-warp CTA holds
  int NC = 0, NG = 0, NF = 0;
  bool fit = false;
  // preference: enough fetchers (a fetcher serialises poll + L2 read per
  // batch), then near groups, then combiners (cheap per batch)
  const int nf_max = std::max(1, env_int("PIPEDP_SDP2_FETCH", 4));
  const int nw_max = std::max(1, std::min(4, env_int("PIPEDP_SDP2_WRITERS", 1)));  // <= 4 progress counters
  const int ng_max = std::max(1, env_int("PIPEDP_SDP2_NEAR_GROUP", 2));
  const int nc_min = std::max(1, env_int("PIPEDP_SDP2_COMB", 2));
  int NWR = 1;
  for (int nf = nf_max; nf >= 1 && !fit; nf = nf > 1 ? nf / 2 : 0) {
    for (int nwr = nw_max; nwr >= 1 && !fit; nwr = nwr > 1 ? nwr / 2 : 0) {
      for (int ng = ng_max; ng >= 1 && !fit; --ng) {
        for (int nc = nc_min; nc >= 1 && !fit; --nc) {
          const int f = remote ? nf : 0, wr = remote ? nwr : 1;
          if (sdp2_warps(NW, ng, nc, f, wr) <= kMaxWarpsV2) {
            NC = nc;
            NG = ng;
            NF = f;
            NWR = wr;
            fit = true;
          }
        }
      }
    }
  }
  if (!fit) return false;
  s.ring_log2 = ceil_log2((uint64_t)R);
  s.a_rem = a_rem;
  s.a_chain = a_chain;
  s.pub_every = std::max(1, env_int("PIPEDP_SDP2_PUB", 4));
  s.n_pre_u = 0;
  s.dom = dom ? 1 : 0;
  for (int64_t j = k - 1; j >= 0 && !dom; --j) {
    if (offs[j] < 64) continue;
    if (offs[j] >= a_chain) break;
    s.pre_u[s.n_pre_u++] = -(int32_t)(offs[j] * (int64_t)vb);
  }
  for (int i = s.n_pre_u; i < kPreUMax; ++i) s.pre_u[i] = 0;
  s.near_warps = NW;
  s.comb_warps = NC;
  s.near_group = NG;
  s.fetchers = std::max(1, NF);
  s.writers = NWR;
  s.j_rem = (int32_t)jr;
  for (int j = 0; j <= NW; ++j) s.near_lo[j] = (int32_t)(jr + (NW ? count * j / NW : 0));
  const size_t smem = sdp_v2_smem(R, ((k - jr) + 3) & ~3ll, vb, NW, NC);
  if (smem > kSmemBudget) return false;
  d->v2 = true;
  d->remote = remote;
  d->small = false;
  d->gfar = false;
  d->warp_kernel = false;
  d->smem = smem;
  d->threads = 32 * sdp2_warps(NW, NG, NC, remote ? NF : 0, NWR);
  d->grid_extra = 0;
  SdpShape& ps = d->shape;  // the producers' view
  ps.n = n;
  ps.k = (int32_t)k;
  ps.a1 = (int32_t)a1;
  ps.a_remote = a_rem;
  ps.remote_warps = 0;
  ps.writers = NWR;
  if (remote) {
    ps.remote_warps = std::min(24, env_int("PIPEDP_SDP_REMOTE_WARPS", 16));
    d->grid_extra = std::min(sm_count() - 1, env_int("PIPEDP_SDP_REMOTE_CTAS", 64));
    d->threads = std::max(d->threads, 32 * ps.remote_warps);
    ps.j_rem = (int32_t)jr;
    ps.rem_look = jr > 0 ? (int32_t)(offs[jr - 1] / 32) : 0;
    const size_t psmem = (size_t)ps.remote_warps * 32 * 8 + 64;
    d->smem = std::max(d->smem, psmem);
  }
  return true;
}

int plan_sdp(int64_t batch, int64_t n, int64_t k, int64_t a1, const int64_t* offsets,
             const int64_t* init, int op, SdpDispatch* d) {
  if (op < 0 || op > 3) return fail(PIPEDP_E_INVALID_PARAMS, "unknown operator kind");
  if (a1 >= (1ll << 27) || k >= (1ll << 24))
    return fail(PIPEDP_ERR_UNSUPPORTED, "a_1=%lld exceeds the 32-bit byte-offset range of the kernels",
                (long long)a1);
  d->op = op;
  d->cluster = false;
  sdp_value_class(op, init, batch * a1, &d->bits, &d->assoc);
  const size_t vb = d->bits / 8;
  SdpShape& s = d->shape;
  s.n = n;
  s.k = (int32_t)k;
  s.a1 = (int32_t)a1;
  s.a_mid = kAMid;
  s.a_remote = 1 << 30;
  s.remote_warps = 0;
  s.writers = 1;
  d->grid_extra = 0;
  d->remote = false;
  const int64_t kpad = (k + 3) & ~3ll;
  // warp-per-instance kernel for batches of small-a_1 instances
  if (batch > 1) {
    const int64_t R = 1ll << ceil_log2((uint64_t)(a1 + 32));
    const size_t per_warp = 2 * R * vb + 2 * kpad * 4;
    if (per_warp <= 16 * 1024) {
      d->warp_kernel = true;
      d->small = a1 < 64;
      d->gfar = false;
      s.ring_log2 = ceil_log2((uint64_t)R);
      s.ring_cover = (int32_t)a1;
      s.mid_warps = s.far_warps = 0;
      d->wpb = (int)std::max<int64_t>(1, std::min<int64_t>(std::max(1, std::min(8, env_int("PIPEDP_SDP_WPB", 8))),
                                                           (96 * 1024) / per_warp));
      d->threads = 32 * d->wpb;
      d->smem = per_warp * d->wpb;
      return PIPEDP_OK;
    }
  }
  d->warp_kernel = false;
  d->small = a1 < 64;
  d->serial = batch == 1 && d->small && k <= 8 && env_int("PIPEDP_SDP_SERIAL", 1) != 0;
  {  // jump-ahead segments (sdp_jump.cuh): a_1 <= 8, an operator whose matrix form is exact
    bool nonneg = true;
    for (int64_t i = 0; i < a1; ++i) nonneg = nonneg && init[i] >= 0;
    const bool ring_ok = op == PIPEDP_OP_MIN || op == PIPEDP_OP_MAX || op == PIPEDP_OP_MODULAR_ADD ||
                         (op == PIPEDP_OP_SATURATING_ADD && nonneg);
    d->jump = batch == 1 && a1 >= 2 && a1 <= 8 && k >= 2 && ring_ok && n - a1 >= 4096 &&
              env_int("PIPEDP_SDP_JUMP", 1) != 0;
  }

  {  // chunks: cells [a1, n) in G <= 2 x SMs chunks (two chunk CTAs share an
     // SM) of L cells, L >= max(4096, 8 a1), L / 32 with <= 3 set bits (each
     // set bit beyond the first costs one matrix product)
    d->chunked = false;
    if (batch == 1 && (op == PIPEDP_OP_MIN || op == PIPEDP_OP_MAX) && a1 >= 64 && a1 <= 8192 &&
        env_int("PIPEDP_SDP_CHUNKED", 1) != 0) {
      // chunk CTAs per SM: two for the generic chunk pipeline; the rank
      // kernel (k <= 4096) fits three when its pair ring is small enough
      // (C2: 293 -> 443 chunks, 3.04 -> 2.96 ms measured)
      const int64_t rank_smem = 8 * (a1 + 160) + 20 * 1024;
      const int per_sm = k <= 4096 && 3 * rank_smem <= 220 * 1024 ? 3 : 2;
      const int64_t slots = (int64_t)per_sm * sm_count();
      const int64_t lmin = std::max<int64_t>(4096, 8 * a1);
      int64_t target = std::max<int64_t>(lmin, (n - a1 + slots - 1) / slots);
      int64_t L = (target + 31) / 32;  // in units of 32 cells
      while (__builtin_popcountll((unsigned long long)L) > 3) ++L;
      L *= 32;
      const int64_t G = (n - a1 + L - 1) / L;
      if (G >= 16) {
        d->chunked = true;
        d->chunk_len = L;
      }
    }
  }
  if (d->small) {
    s.ring_log2 = ceil_log2((uint64_t)(a1 + 128));
    s.ring_cover = (int32_t)a1;
    s.mid_warps = s.far_warps = 0;
    d->gfar = false;
    d->threads = 32;
    d->smem = sdp_cta_smem(1ll << s.ring_log2, kpad, vb);
    return PIPEDP_OK;
  }
  d->v2 = false;
  if (batch == 1 && d->assoc && d->bits == 32 && op != PIPEDP_OP_SATURATING_ADD &&
      env_int("PIPEDP_SDP_CLUSTER", 1) != 0) {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        pipedp_cluster::plan(offsets, (int32_t)k, (int32_t)a1, n, op, dev, &d->cplan)) {
      d->cluster = true;
      return PIPEDP_OK;
    }
    (void)cudaGetLastError();
  }
  if (batch == 1 && d->assoc && !(op == PIPEDP_OP_MODULAR_ADD && d->bits == 64) &&
      env_int("PIPEDP_SDP_V2", 1) != 0 && plan_sdp_v2(n, k, a1, offsets, d))
    return PIPEDP_OK;
  // offset counts per stage (max over the batch sizes the stages)
  int64_t jf_max = 0, jr_max = 0;
  for (int64_t b = 0; b < batch; ++b) {
    int64_t jf = 0, jr = 0;
    for (int64_t j = 0; j < k; ++j) {
      jf += offsets[b * k + j] >= kAMid;
      jr += offsets[b * k + j] >= kARemote;
    }
    jf_max = std::max(jf_max, jf);
    jr_max = std::max(jr_max, jr);
  }
  // multi-CTA: one large associative instance with enough remote work
  const int64_t nb = (n - a1 + 31) / 32;
  d->remote = batch == 1 && d->assoc && jr_max >= 128 && nb >= 256 &&
              env_int("PIPEDP_SDP_MULTI", 1) != 0;
  s.mid_warps = env_int("PIPEDP_SDP_MID_WARPS", 4);
  if (d->remote) {
    const int a_rem = std::max(kAMid, env_int("PIPEDP_SDP_AREMOTE", kARemote));
    s.a_remote = a_rem;
    s.ring_cover = a_rem;
    s.ring_log2 = ceil_log2((uint64_t)(a_rem + 512));
    d->gfar = false;
    s.far_warps = (int32_t)std::min<int64_t>(16, std::max<int64_t>(1, (jf_max - jr_max + 47) / 48));
    s.remote_warps = env_int("PIPEDP_SDP_REMOTE_WARPS", 8);
    {
      int64_t jr0 = 0;
      for (int64_t j = 0; j < k; ++j) jr0 += offsets[j] >= a_rem;  // one instance (batch == 1)
      s.j_rem = (int32_t)jr0;
      s.rem_look = jr0 > 0 ? (int32_t)(offsets[jr0 - 1] / 32) : 0;
    }
    d->grid_extra = std::min(sm_count() - 1, env_int("PIPEDP_SDP_REMOTE_CTAS", 32));
    d->smem = sdp_cta_smem(1ll << s.ring_log2, kpad, vb);
  } else {
    const int64_t r_full = 1ll << ceil_log2((uint64_t)(a1 + 512));
    const size_t smem_full = sdp_cta_smem(r_full, kpad, vb);
    if (smem_full <= kSmemBudget) {
      d->gfar = false;
      s.ring_log2 = ceil_log2((uint64_t)r_full);
      s.ring_cover = (int32_t)a1;
      d->smem = smem_full;
    } else {
      d->gfar = true;
      s.ring_log2 = ceil_log2((uint64_t)(kAMid + 512));
      s.ring_cover = kAMid;
      d->smem = sdp_cta_smem(1ll << s.ring_log2, kpad, vb);
      if (d->smem > 227 * 1024)
        return fail(PIPEDP_ERR_UNSUPPORTED, "k=%lld offsets exceed shared memory", (long long)k);
    }
    s.far_warps = (int32_t)std::min<int64_t>(std::max(1, std::min(19, env_int("PIPEDP_SDP_FAR_MAX", 19))),
                                             std::max<int64_t>(1, (jf_max + 47) / 48));  // <= 32 warps
  }
  d->threads = 32 * sdp_warps_for_roles(s.mid_warps + s.far_warps + 1);
  d->threads = std::max(d->threads, 32 * s.remote_warps);
  return PIPEDP_OK;
}

template <int OP, typename T, bool SMALL, bool ASSOC, bool GFAR>
int launch_cta(const SdpDispatch& d, int64_t batch, const int64_t* offs, const int64_t* init,
               int64_t* out, cudaStream_t st) {
  auto kern = sdp_pipeline_cta<OP, T, SMALL, ASSOC, GFAR>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem));
  kern<<<(unsigned)batch, d.threads, d.smem, st>>>(d.shape, offs, init, out);
  CK(cudaGetLastError());
  return PIPEDP_OK;
}

template <int OP, typename T>
int launch_multi(const SdpDispatch& d, const int64_t* offs, const int64_t* init, int64_t* out,
                 const SdpRemote& rm, cudaStream_t st) {
  auto kern = sdp_pipeline_multi<OP, T, false>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem));
  SdpShape shape = d.shape;
  void* args[] = {(void*)&shape, (void*)&offs, (void*)&init, (void*)&out, (void*)&rm};
  CK(cudaLaunchCooperativeKernel((void*)kern, dim3(1 + d.grid_extra), dim3(d.threads), args, d.smem, st));
  return PIPEDP_OK;
}

template <int OP, typename T, bool SMALL, bool ASSOC>
int launch_warp(const SdpDispatch& d, int64_t batch, const int64_t* offs, const int64_t* init,
                int64_t* out, cudaStream_t st) {
  auto kern = sdp_batch_warp<OP, T, SMALL, ASSOC>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem));
  const int64_t grid = (batch + d.wpb - 1) / d.wpb;
  kern<<<(unsigned)grid, d.threads, d.smem, st>>>(d.shape, batch, offs, init, out);
  CK(cudaGetLastError());
  return PIPEDP_OK;
}

template <int OP, typename T>
int launch_v2(const SdpDispatch& d, const int64_t* offs, const int64_t* init, int64_t* out,
              const SdpRemote& rm, cudaStream_t st) {
  if (!d.remote) {
    auto kern = sdp_v2_cta<OP, T>;
    CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem));
    kern<<<1, d.threads, d.smem, st>>>(d.s2, offs, init, out);
    CK(cudaGetLastError());
    return PIPEDP_OK;
  }
  auto kern = sdp_v2_multi<OP, T>;
  CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)d.smem));
  SdpV2Shape s2 = d.s2;
  SdpShape ps = d.shape;
  void* args[] = {(void*)&s2, (void*)&ps, (void*)&offs, (void*)&init, (void*)&out, (void*)&rm};
  CK(cudaLaunchCooperativeKernel((void*)kern, dim3(1 + d.grid_extra), dim3(d.threads), args, d.smem, st));
  return PIPEDP_OK;
}

template <int OP>
int launch_jump(const SdpDispatch& d, const int64_t* offs, const int64_t* init, int64_t* out, cudaStream_t st) {
  const int64_t nseg = (d.shape.n - d.shape.a1 + (1 << kJumpLog2L) - 1) >> kJumpLog2L;
  const unsigned grid = (unsigned)((nseg + kJumpThreads - 1) / kJumpThreads);
  switch (d.shape.a1) {
#define PIPEDP_JUMP_CASE(A) \
  case A: sdp_jump<OP, A><<<grid, kJumpThreads, 0, st>>>(d.shape.n, d.shape.k, offs, init, out); break;
    PIPEDP_JUMP_CASE(2)
    PIPEDP_JUMP_CASE(3)
    PIPEDP_JUMP_CASE(4)
    PIPEDP_JUMP_CASE(5)
    PIPEDP_JUMP_CASE(6)
    PIPEDP_JUMP_CASE(7)
    PIPEDP_JUMP_CASE(8)
#undef PIPEDP_JUMP_CASE
    default: return fail(PIPEDP_E_INVALID_PARAMS, "sdp_jump: a_1 = %d", d.shape.a1);
  }
  CK(cudaGetLastError());
  return PIPEDP_OK;
}

template <int OP, typename T, bool ASSOC>
int launch_sdp_t(const SdpDispatch& d, int64_t batch, const int64_t* offs, const int64_t* init,
                 int64_t* out, const SdpRemote& rm, cudaStream_t st) {
  if (ASSOC && d.method != 0) {  // the paper's comparison methods (one instance, int64)
    if (d.method == 1) {
      // the last a_1 + 1 cells in shared memory when they fit (Table I bucket 1)
      // the last a_1 + 1 cells in shared memory when they fit -- as 4-byte
      // words for a 32-bit value class (Table I buckets 1, 2) -- else operands
      // through L2 (a single SM's L2 bandwidth bounds that path)
      const int64_t a1 = d.shape.a1;
      const size_t ring64 = sizeof(int64_t) * (size_t)(a1 + 1), ring32 = sizeof(int32_t) * (size_t)(a1 + 1);
      const bool few = (d.shape.k + 1023) / 1024 <= 8;  // offsets per thread: 8 or 32 register slots
      auto ring_launch = [&](auto kern, size_t bytes) -> int32_t {
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
        kern<<<1, 1024, bytes, st>>>(d.shape.n, d.shape.k, offs, init, out, (int32_t)(a1 + 1));
        return PIPEDP_OK;
      };
      if (ring64 <= 200 * 1024) {
        TRY(few ? ring_launch(sdp_tournament<OP, int64_t, 8>, ring64) : ring_launch(sdp_tournament<OP, int64_t, 32>, ring64));
      } else if (d.vals32 && ring32 <= 200 * 1024) {
        TRY(few ? ring_launch(sdp_tournament<OP, int32_t, 8>, ring32) : ring_launch(sdp_tournament<OP, int32_t, 32>, ring32));
      } else {
        sdp_tournament<OP, void><<<1, 1024, 0, st>>>(d.shape.n, d.shape.k, offs, init, out, 1);
      }
    }
    else sdp_naive<OP><<<1, 1024, 0, st>>>(d.shape.n, d.shape.k, offs, init, out);
    CK(cudaGetLastError());
    return PIPEDP_OK;
  }
  if (ASSOC && d.cluster) {
    CK(pipedp_cluster::launch(d.cplan, offs, init, out, st));
    return PIPEDP_OK;
  }
  if (ASSOC && d.v2 && !(OP == kModAdd && sizeof(T) == 8)) return launch_v2<OP, T>(d, offs, init, out, rm, st);
  if (d.jump) return launch_jump<OP>(d, offs, init, out, st);
  if (d.serial) {
    sdp_serial_thread<OP, T><<<1, 32, 0, st>>>(d.shape.n, d.shape.k, offs, init, out);
    CK(cudaGetLastError());
    return PIPEDP_OK;
  }
  if (d.warp_kernel) {
    return d.small ? launch_warp<OP, T, true, ASSOC>(d, batch, offs, init, out, st)
                   : launch_warp<OP, T, false, ASSOC>(d, batch, offs, init, out, st);
  }
  if (d.small) return launch_cta<OP, T, true, ASSOC, false>(d, batch, offs, init, out, st);
  if (ASSOC && d.remote) return launch_multi<OP, T>(d, offs, init, out, rm, st);
  return d.gfar ? launch_cta<OP, T, false, ASSOC, true>(d, batch, offs, init, out, st)
                : launch_cta<OP, T, false, ASSOC, false>(d, batch, offs, init, out, st);
}

int launch_sdp(const SdpDispatch& d, int64_t batch, const int64_t* offs, const int64_t* init,
               int64_t* out, const SdpRemote& rm, cudaStream_t st) {
  switch (d.op) {
    case PIPEDP_OP_MIN:
      return d.bits == 32 ? launch_sdp_t<kMin, int32_t, true>(d, batch, offs, init, out, rm, st)
                          : launch_sdp_t<kMin, int64_t, true>(d, batch, offs, init, out, rm, st);
    case PIPEDP_OP_MAX:
      return d.bits == 32 ? launch_sdp_t<kMax, int32_t, true>(d, batch, offs, init, out, rm, st)
                          : launch_sdp_t<kMax, int64_t, true>(d, batch, offs, init, out, rm, st);
    case PIPEDP_OP_MODULAR_ADD:
      return d.bits == 32 ? launch_sdp_t<kModAdd, int32_t, true>(d, batch, offs, init, out, rm, st)
                          : launch_sdp_t<kModAdd, int64_t, true>(d, batch, offs, init, out, rm, st);
    default:
      return d.assoc ? launch_sdp_t<kSatAdd, int64_t, true>(d, batch, offs, init, out, rm, st)
                     : launch_sdp_t<kSatAdd, int64_t, false>(d, batch, offs, init, out, rm, st);
  }
}

const char* sdp_kernel_name(const SdpDispatch& d) {
  if (d.method == 1 && d.assoc) return "sdp_tournament";
  if (d.method == 2 && d.assoc) return "sdp_naive";
  if (d.cluster) return "sdp_cluster_kernel";
  if (d.jump) return "sdp_jump";
  if (d.serial) return "sdp_serial_thread";
  if (d.v2) return d.remote ? "sdp_v2_multi" : "sdp_v2_cta";
  if (d.warp_kernel) return "sdp_batch_warp";
  if (d.small) return "sdp_pipeline_cta[chain]";
  if (d.remote) return "sdp_pipeline_multi";
  return d.gfar ? "sdp_pipeline_cta[far-hbm]" : "sdp_pipeline_cta[ring]";
}

}  // namespace

constexpr size_t kRemoteBytes = kRemSlots * 32 * sizeof(int64_t) + kRemSlots * sizeof(int) + 64;

// Host tables from this size on are pre-faulted while the kernels run and (for
// the 32-bit value class) copied out narrowed.
static const size_t kHostCopyBig = (size_t)std::max(1, env_int("PIPEDP_HOST_COPY_BIG_KB", 2048)) << 10;

// int64 -> int32 for a table whose values are proven to fit (the host widens
// it back while copying out: half the device -> host bytes).
__global__ void narrow_i64_i32(const int64_t* __restrict__ src, int32_t* __restrict__ dst, int64_t count) {
  const int64_t pairs = count / 2;
  const int4* s2 = reinterpret_cast<const int4*>(src);
  int2* d2 = reinterpret_cast<int2*>(dst);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < pairs; i += (int64_t)gridDim.x * blockDim.x) {
    const int4 v = s2[i];  // two int64: (x, y) and (z, w) little-endian halves
    d2[i] = make_int2(v.x, v.z);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (count & 1)) dst[count - 1] = (int32_t)src[count - 1];
}

// Copy an int64 device table out through an int32 staging copy (W->buffer slot).
static int32_t d2h_narrowed(pipedp_host::Workspace* W, int slot, int64_t* host, const int64_t* dev, int64_t count,
                            cudaStream_t st = nullptr) {
  if (!st) st = W->stream;
  void* tmp = nullptr;
  CK(W->buffer(slot, sizeof(int32_t) * (size_t)count + 16, &tmp));
  narrow_i64_i32<<<(unsigned)std::min<int64_t>(4 * 148, (count / 2 + 255) / 256 + 1), 256, 0, st>>>(
      dev, static_cast<int32_t*>(tmp), count);
  CK(cudaGetLastError());
  CK(W->d2h_widen(host, static_cast<const int32_t*>(tmp), (size_t)count, st));
  return PIPEDP_OK;
}

struct pipedp_sdp_plan {
  int device;
  int64_t batch, n, k, a1;
  SdpDispatch d;
  // chunked mode (d.chunked): G chunks of Lc cells, each an instance of n_i =
  // a1 + Lc cells solved by the batch dispatch dc
  int64_t G = 0, Lc = 0, n_i = 0;
  int32_t W = 0;                       // 64-bit words per boolean matrix row
  SdpDispatch dc{};
  unsigned long long* d_bm = nullptr;  // X, XT, Z, ZT: [64 W][W] each
  unsigned long long* d_q = nullptr;   // Q = M^Lc kept while Q^16 is formed
  int64_t* d_E = nullptr;              // two state vectors [64 W]
  int64_t* d_cinit = nullptr;          // [G][a1] chunk preset cells
  int64_t* d_offs_rep = nullptr;       // [G][k]
  int64_t* d_pad = nullptr;            // [G][n_i] chunk tables
  int32_t* d_perm = nullptr;           // batch warp kernel: instance order (dominance-form ones first)
  int64_t* d_offsets;  // device copy of the offsets, int64 [batch*k]
  void* d_remote;      // multi-CTA workspace: partial slots | ready flags | published
  int32_t* d_obg;      // remote producers: offsets as HBM-table byte offsets
  // chunked min / max on 16-bit ranks (sdp_rank.cu); null: the generic chunk batch
  pipedp_rank::ChunkRankParams* rank = nullptr;
  int rank_threads = 0;
  size_t rank_smem = 0;
  int64_t* d_sorted = nullptr;  // [a1] init ascending: rank -> value
  // batched min / max: instances perm[0, n_dom) take the dominance kernel
  // (sdp_batch_dom.cu), the rest sdp_batch_warp
  int64_t n_dom = 0;
  pipedp_bdom::DomInfo* d_dinfo = nullptr;
  // the fallback instances run beside the dominance kernel (fork / join)
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // phase timing of the chunked mode (pipedp_sdp_plan_set_timing): events at
  // the start, after the matrix powers, after the entry-state chain, after
  // the chunk batch; accumulated per phase until read
  bool timing = false;
  cudaEvent_t ev_phase[4] = {nullptr, nullptr, nullptr, nullptr};
  double phase_ms[3] = {0, 0, 0};
  int64_t phase_runs = 0;
  bool phase_pending = false;
};

// ================================================================== MCM ===
namespace {

struct McmDispatch {
  int kernel;  // PIPEDP_MCM_WAVEFRONT / SMEM / TOURNAMENT / TILED
  int tile;    // tiled kernel: tile edge (32 or 64)
  int bits;    // 32 or 64 (first attempt)
  int threads;
  size_t smem32, smem64;
};

int mcm_max_dim(const int64_t* dims, int64_t len) {
  int64_t m = 1;
  for (int64_t i = 0; i < len; ++i) m = std::max(m, dims[i]);
  return (int)std::min<int64_t>(m, INT_MAX);
}

size_t mcm_smem_bytes(int64_t n, size_t vb) {
  const int64_t cc = n * (n + 1) / 2;
  return ((cc + 1 + 3) & ~3ll) * vb + (n + 1 + 3) * 4;
}

int plan_mcm(int64_t batch, int64_t n, const int64_t* dims, int kernel, McmDispatch* d) {
  int max_dim = 1;
  for (int64_t b = 0; b < batch; ++b) max_dim = std::max(max_dim, mcm_max_dim(dims + b * (n + 1), n + 1));
  d->bits = max_dim <= 1290 ? 32 : 64;  // max_dim^3 < 2^31
  d->smem32 = mcm_smem_bytes(n, 4);
  d->smem64 = mcm_smem_bytes(n, 8);
  if (kernel == PIPEDP_MCM_AUTO) {
    const size_t need = d->bits == 32 ? d->smem32 : d->smem64;
    const bool fits = need <= kSmemBudget;
    kernel = (fits && (batch > 1 || n <= 160)) ? PIPEDP_MCM_SMEM : PIPEDP_MCM_WAVEFRONT;
    if (!fits && batch > 1) kernel = PIPEDP_MCM_WAVEFRONT;
    if (kernel == PIPEDP_MCM_WAVEFRONT && batch == 1 && d->bits == 32 &&
        env_int("PIPEDP_MCM_TILED", 1) != 0)
      kernel = PIPEDP_MCM_TILED;
  }
  if (kernel == PIPEDP_MCM_TILED && batch > 1)
    return fail(PIPEDP_E_INVALID_PARAMS, "the tiled kernel solves one instance at a time");
  d->tile = (n <= env_int("PIPEDP_MCM_T32_MAXN", 2048)) ? 32 : 64;
  if (kernel == PIPEDP_MCM_TILED && (n + d->tile - 1) / d->tile >= 65535)
    return fail(PIPEDP_ERR_UNSUPPORTED, "n=%lld too large for the tiled MCM kernel", (long long)n);
  if (kernel == PIPEDP_MCM_SMEM && d->smem64 > 227 * 1024 && d->smem32 > 227 * 1024)
    return fail(PIPEDP_ERR_UNSUPPORTED, "n=%lld too large for the shared-memory MCM kernel",
                (long long)n);
  if (kernel == PIPEDP_MCM_SMEM && d->bits == 64 && d->smem64 > 227 * 1024)
    return fail(PIPEDP_ERR_UNSUPPORTED, "n=%lld too large for the 64-bit shared-memory MCM kernel",
                (long long)n);
  if ((kernel == PIPEDP_MCM_TOURNAMENT) && batch > 1)
    return fail(PIPEDP_E_INVALID_PARAMS, "the tournament kernel solves one instance at a time");
  if (kernel < PIPEDP_MCM_AUTO || kernel > PIPEDP_MCM_TILED)
    return fail(PIPEDP_E_INVALID_PARAMS, "unknown MCM kernel %d", kernel);
  d->kernel = kernel;
  d->threads = n <= 64 ? 128 : (n <= 256 ? 256 : 512);
  return PIPEDP_OK;
}

}  // namespace

struct pipedp_mcm_plan {
  int device;
  int64_t batch, n, cc;
  McmDispatch d;
  int32_t* d_p;       // dims as int32 [batch*(n+1)] (validated <= 1e6)
  int64_t* d_dims;    // dims int64 (tournament)
  uint32_t* d_v32;    // wavefront 32-bit value table [cc+1]
  int64_t* d_chunk_base;
  int* d_done;
  unsigned long long* d_next;
  int* d_overflow;
  int* h_overflow;    // pinned
  int64_t total_chunks;
  int launches;
  int last_bits;      // 0: an async execute not resolved yet (mcm_resolve)
  int gate;           // overflow bits the next launch is conditional on (0: always)
  bool pending;       // last execute ran with on-device reruns; flag not read yet
  cudaEvent_t ev_done;
  int64_t maxd3;      // max_dim^3 over the plan's instances
  bool packed_now;    // this execute's tiled launch uses them
  // tiled kernel
  int32_t* d_pp;                 // dims, zero padded to N*T + 2
  uint32_t* d_tiles;
  unsigned long long* d_keys;
  int* d_tile_flags;             // tile_done | far_count
  unsigned long long* d_tasks;
  int64_t ntasks;
  int32_t N;
  int tiled_grid;
};

namespace {

int mcm_wave_launch(pipedp_mcm_plan* P, int bits, int64_t* cells, int64_t* split, cudaStream_t st) {
  // one dataflow wavefront per instance (a batch runs them back to back on the
  // stream; the done/next/value scratch is reset for each)
  const int64_t n = P->n, cc = P->cc;
  int dev = 0, sms = 148;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int threads = 256;
  int64_t grid = std::min<int64_t>((int64_t)sms * 8, (P->total_chunks + 7) / 8);
  grid = std::max<int64_t>(grid, 1);
  for (int64_t b = 0; b < P->batch; ++b) {
    int64_t* cb = cells + b * (cc + 1);
    int64_t* sb = split + b * (cc + 1);
    const int32_t* pb = P->d_p + b * (n + 1);
    CK(cudaMemsetAsync(P->d_done, 0, sizeof(int) * std::max<int64_t>(P->total_chunks, 1), st));
    CK(cudaMemsetAsync(P->d_next, 0, sizeof(unsigned long long), st));
    CK(cudaMemsetAsync(cb, 0, sizeof(int64_t) * (n + 1), st));
    CK(cudaMemsetAsync(sb, 0, sizeof(int64_t) * (n + 1), st));
    McmWave W{n, P->total_chunks, P->d_chunk_base, P->d_done, P->d_next};
    if (bits == 32) {
      CK(cudaMemsetAsync(P->d_v32, 0, sizeof(uint32_t) * (n + 1), st));
      mcm_wavefront<uint32_t><<<(unsigned)grid, threads, 0, st>>>(W, pb, P->d_v32, cb, sb, P->d_overflow, P->gate);
    } else {
      mcm_wavefront<int64_t><<<(unsigned)grid, threads, 0, st>>>(W, pb, cb, cb, sb, P->d_overflow, P->gate);
    }
    CK(cudaGetLastError());
  }
  return PIPEDP_OK;
}

int mcm_tiled_launch(pipedp_mcm_plan* P, int64_t* cells, int64_t* split, cudaStream_t st) {
  const int64_t n = P->n, N = P->N, ntiles = N * (N + 1) / 2;
  const int64_t TC = (int64_t)P->d.tile * P->d.tile;
  CK(cudaMemsetAsync(P->d_keys, 0xFF, sizeof(unsigned long long) * ntiles * TC, st));
  CK(cudaMemsetAsync(P->d_tile_flags, 0, sizeof(int) * 2 * ntiles, st));
  CK(cudaMemsetAsync(P->d_next, 0, sizeof(unsigned long long), st));
  CK(cudaMemsetAsync(cells, 0, sizeof(int64_t) * (n + 1), st));
  CK(cudaMemsetAsync(split, 0, sizeof(int64_t) * (n + 1), st));
  McmTiled S{n, (int32_t)N, P->ntasks, P->d_pp, P->d_tiles, P->d_keys, P->d_tile_flags,
             P->d_tile_flags + ntiles, P->d_tasks, P->d_next, cells, split, P->d_overflow,
             env_int("PIPEDP_MCM_BLOCKED", 0) ? 1 : env_int("PIPEDP_MCM_NEAR", 2), P->packed_now ? 1 : 0,
             P->gate};
  if (P->d.tile == 32) {
    CK(cudaFuncSetAttribute(t32::mcm_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)t32::kTiledSmemBytes));
    t32::mcm_tiled_kernel<<<(unsigned)P->tiled_grid, kTiledThreads, t32::kTiledSmemBytes, st>>>(S);
  } else {
    CK(cudaFuncSetAttribute(t64::mcm_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)t64::kTiledSmemBytes));
    t64::mcm_tiled_kernel<<<(unsigned)P->tiled_grid, kTiledThreads, t64::kTiledSmemBytes, st>>>(S);
  }
  CK(cudaGetLastError());
  return PIPEDP_OK;
}

// Task list of the tiled kernel, ordered by readiness (see mcm_tiled.cuh):
// far task (I, J, K) at level L = max(K-I, J-K) (its inputs are tiles of
// levels <= L), its level's tasks by tile distance Delta = J - I ascending; the
// near task of a tile at level Delta - 1, right after the far tasks of the
// tiles of distance Delta (its own last far tasks) and before the far tasks
// that feed farther tiles -- the critical chain (near Delta-1 -> the two last
// far tasks -> near Delta) is not queued behind a level's whole far work.
std::vector<unsigned long long> mcm_tiled_tasks(int N) {
  std::vector<unsigned long long> out;
  for (int I = 0; I < N; ++I) out.push_back(tiled_task(kTaskDiag, I, I, 0));
  for (int L = 0; L + 1 < N; ++L) {
    // far tasks of level L (L >= 1) for tiles of distance D in [L+1, 2L], D ascending;
    // the near tasks of distance L+1 after the D = L+1 group
    for (int D = L + 1; D <= 2 * L + 1 && D < N; ++D) {
      if (L >= 1 && D <= 2 * L)
        for (int I = 0; I + D < N; ++I) {
          const int J = I + D;
          // the two K of level L (J - L < I + L) in one task, except for the
          // tiles whose near task comes next (D = L + 1): those two run in
          // parallel, they are the critical chain; D = 2L: one K
          if (D == 2 * L) {
            out.push_back(tiled_task(kTaskFar, I, J, I + L));
          } else if (D == L + 1) {
            out.push_back(tiled_task(kTaskFar, I, J, I + L));
            out.push_back(tiled_task(kTaskFar, I, J, J - L));
          } else {
            out.push_back(tiled_task(kTaskFar2, I, J, J - L));
          }
        }
      if (D == L + 1)
        for (int I = 0; I + D < N; ++I) out.push_back(tiled_task(kTaskNear, I, I + D, 0));
    }
  }
  return out;
}

size_t mcm_square_bytes(int64_t n, size_t vb) {
  const int64_t P = n + 1;
  return (size_t)(P * P + 1) * vb + (size_t)(n + 1 + 4) * 4;
}

// CTAs of a square / triangle batch launch: one per instance, or for a gated
// rerun (usually a no-op) a few per SM looping over the instances
unsigned mcm_grid(const pipedp_mcm_plan* P) {
  return (unsigned)(P->gate ? std::min<int64_t>(P->batch, 4 * (int64_t)sm_count()) : P->batch);
}

int mcm_smem_launch(pipedp_mcm_plan* P, int bits, int64_t* cells, int64_t* split, cudaStream_t st) {
  const int64_t n = P->n;
  const size_t sq = mcm_square_bytes(n, bits / 8);
  if (bits == 32 && P->packed_now && n <= pipedp_mcmb::kMaxN && env_int("PIPEDP_MCM_BATCH_WARP", 1) != 0) {
    // one warp per instance, packed keys (mcm_batch.cu)
    CK(pipedp_mcmb::launch((int32_t)n, P->batch, P->d_dims, cells, split, P->d_overflow, st));
    return PIPEDP_OK;
  }
  if (sq <= kSmemBudget && env_int("PIPEDP_MCM_SQUARE", 1) != 0) {
    // row-major square table: incremental operand addresses (mcm_smem_square)
    // two warps for n <= 96: the short diagonals keep them busy (C5a: 3.96 ->
    // 3.19 ms against four warps); more CTAs fit an SM
    const int thr = std::max(32, std::min(128, env_int("PIPEDP_MCM_SQ_THREADS", n <= 96 ? 64 : 128))) / 32 * 32;
    if (bits == 32 && P->packed_now && n <= 64) {
      CK(cudaFuncSetAttribute(mcm_smem_square<uint32_t, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sq));
      mcm_smem_square<uint32_t, true><<<mcm_grid(P), thr, sq, st>>>((int32_t)n, P->batch, P->d_dims, cells,
                                                                            split, P->d_overflow, P->gate);
    } else if (bits == 32) {
      CK(cudaFuncSetAttribute(mcm_smem_square<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sq));
      mcm_smem_square<uint32_t><<<mcm_grid(P), thr, sq, st>>>((int32_t)n, P->batch, P->d_dims, cells,
                                                                      split, P->d_overflow, P->gate);
    } else {
      CK(cudaFuncSetAttribute(mcm_smem_square<int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sq));
      mcm_smem_square<int64_t><<<mcm_grid(P), thr, sq, st>>>((int32_t)n, P->batch, P->d_dims, cells,
                                                                     split, P->d_overflow, P->gate);
    }
    CK(cudaGetLastError());
    return PIPEDP_OK;
  }
  if (bits == 32) {
    CK(cudaFuncSetAttribute(mcm_smem_cta<uint32_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)P->d.smem32));
    mcm_smem_cta<uint32_t><<<mcm_grid(P), P->d.threads, P->d.smem32, st>>>(
        n, P->batch, P->d_dims, cells, split, P->d_overflow, P->gate);
  } else {
    CK(cudaFuncSetAttribute(mcm_smem_cta<int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)P->d.smem64));
    mcm_smem_cta<int64_t><<<mcm_grid(P), P->d.threads, P->d.smem64, st>>>(
        n, P->batch, P->d_dims, cells, split, P->d_overflow, P->gate);
  }
  CK(cudaGetLastError());
  return PIPEDP_OK;
}

int mcm_execute(pipedp_mcm_plan* P, int64_t* cells, int64_t* split, cudaStream_t st) {
  P->launches = 0;
  if (P->d.kernel == PIPEDP_MCM_TOURNAMENT) {  // the paper's method, diagonal-parallel (mcm_tournament.cu)
    CK(pipedp_tour::launch(P->n, P->d_dims, cells, split, reinterpret_cast<unsigned*>(P->d_overflow + 2), st));
    P->launches = 1;
    P->last_bits = 64;
    return PIPEDP_OK;
  }
  int bits = P->d.bits;
  // packed keys: the 64-wide tiles' far tasks (ALU-bound; the 32-wide ones are
  // latency-bound and keep the plain fold) and the n <= 64 square-table batches
  const bool tiled_pk = P->d.kernel == PIPEDP_MCM_TILED && P->d.tile == 64 && P->maxd3 < (int64_t)kMcmPackedLimit;
  // (n <= 64: the warp-per-instance kernel mcm_batch_warp, or with
  // PIPEDP_MCM_BATCH_WARP=0 the square-table CTAs' packed fold)
  const bool square_pk = P->d.kernel == PIPEDP_MCM_SMEM && P->d.bits == 32 && P->n <= 64 &&
                         P->maxd3 < (1ll << 24) && env_int("PIPEDP_MCM_PACKED_SQUARE", 1) != 0;
  P->packed_now = (tiled_pk || square_pk) && env_int("PIPEDP_MCM_PACKED", 1) != 0;
  int kernel = P->d.kernel;  // this execute's kernel (the plan itself is never changed)
  // 64-bit fallback of this plan's kernel: one launch (asynchronous reruns), or
  // an instance-by-instance wavefront for a batch whose 64-bit table does not
  // fit shared memory (those few shapes keep the host round trip)
  const int kernel64 = kernel == PIPEDP_MCM_SMEM && P->d.smem64 > 227 * 1024 ? PIPEDP_MCM_WAVEFRONT
                       : kernel == PIPEDP_MCM_TILED                          ? PIPEDP_MCM_WAVEFRONT
                                                                             : kernel;
  auto launch = [&](int kern, int b, int gate) -> int32_t {
    P->gate = gate;
    int32_t rc;
    if (kern == PIPEDP_MCM_SMEM) rc = mcm_smem_launch(P, b, cells, split, st);
    else if (kern == PIPEDP_MCM_TILED && b == 32) rc = mcm_tiled_launch(P, cells, split, st);
    else rc = mcm_wave_launch(P, b, cells, split, st);
    P->gate = 0;
    P->launches += kern == PIPEDP_MCM_WAVEFRONT ? (int)P->batch : 1;
    return rc;
  };
  CK(cudaMemsetAsync(P->d_overflow, 0, sizeof(int), st));
  if (bits == 64) {
    TRY(launch(kernel, 64, 0));
    P->last_bits = 64;
    P->pending = false;
    return PIPEDP_OK;
  }
  if (!(kernel64 == PIPEDP_MCM_WAVEFRONT && P->batch > 1)) {
    // no host round trip: the reruns are launched behind the attempt and do
    // their work only if it raised their overflow bit (mcm_gated_off), so the
    // device plan stays asynchronous (and CUDA-graph capturable)
    const bool packed = P->packed_now;
    TRY(launch(kernel, 32, 0));
    if (packed) {  // bit 2: a packed key could wrap -> the unpacked fold
      P->packed_now = false;
      const int32_t rc = launch(kernel, 32, 2);
      P->packed_now = packed;
      TRY(rc);
    }
    TRY(launch(kernel64, 64, 1));  // bit 1: a value reached 2^30 -> exact int64
    if (!P->ev_done) CK(cudaEventCreateWithFlags(&P->ev_done, cudaEventDisableTiming));
    CK(cudaEventRecord(P->ev_done, st));
    P->last_bits = 0;
    P->pending = true;
    return PIPEDP_OK;
  }
  for (;;) {
    CK(cudaMemsetAsync(P->d_overflow, 0, sizeof(int), st));
    TRY(launch(kernel, bits, 0));
    P->last_bits = bits;
    P->pending = false;
    if (bits == 64) return PIPEDP_OK;
    CK(cudaMemcpyAsync(P->h_overflow, P->d_overflow, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (*P->h_overflow == 0) return PIPEDP_OK;
    if (*P->h_overflow == 2 && P->packed_now) {  // a cell reached 2^25: redo with unpacked far folds
      P->packed_now = false;
      continue;
    }
    bits = 64;  // a value reached 2^30: redo exactly in 64-bit
    kernel = kernel64;
  }
}

// After an asynchronous execute: which attempt's output stands (waits for the
// execute; the host-buffer path and describe() need it).
int32_t mcm_resolve(pipedp_mcm_plan* P) {
  if (!P->pending) return PIPEDP_OK;
  CK(cudaEventSynchronize(P->ev_done));
  int f = 0;
  CK(cudaMemcpy(&f, P->d_overflow, sizeof(int), cudaMemcpyDeviceToHost));
  P->last_bits = (f & 1) ? 64 : 32;
  if (f & 2) P->packed_now = false;
  P->pending = false;
  return PIPEDP_OK;
}

}  // namespace

// ====================================================================== API ===
extern "C" {

const char* pipedp_last_error(void) { return g_last_error.c_str(); }
const char* pipedp_version(void) { return "pipedp-b200 0.1 (sm_100a)"; }
int32_t pipedp_device_count(void) { return usable_devices(); }

int32_t pipedp_sdp_validate(const int64_t* offsets, int64_t k, int64_t init_len, int64_t n) {
  return validate_sdp(offsets, k, init_len, n);
}

int32_t pipedp_mcm_validate(const int64_t* dims, int64_t dims_len) {
  return validate_mcm(dims, dims_len);
}

uint64_t pipedp_table_digest(const int64_t* cells, int64_t count) {  // table.cpp:12-25
  uint64_t h = 14695981039346656037ull;
  auto mix = [&](uint64_t v) {
    for (int b = 0; b < 8; ++b) {
      h ^= (v >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  };
  mix((uint64_t)count);
  for (int64_t i = 0; i < count; ++i) mix((uint64_t)cells[i]);
  return h;
}

// generate.cpp:21-47 -- same draws from the same std::mt19937_64 stream.
int32_t pipedp_generate_sdp(int64_t n, int64_t k, int32_t op, uint64_t seed, int32_t consecutive,
                            int64_t a1_cap, int64_t* offsets_out, int64_t* init_out,
                            int64_t init_cap, int64_t* a1_out) {
  (void)op;
  if (k < 1) return fail(PIPEDP_E_INVALID_PARAMS, "k must be >= 1");
  std::mt19937_64 rng(seed);
  auto bounded = [&](int64_t lo, int64_t hi) {
    return lo + (int64_t)(rng() % (uint64_t)(hi - lo + 1));
  };
  std::vector<int64_t> offs;
  if (consecutive) {
    for (int64_t a = k; a >= 1; --a) offs.push_back(a);
  } else {
    const int64_t cap = a1_cap > 0 ? a1_cap : 2 * k;
    if (cap < k) return fail(PIPEDP_E_INVALID_PARAMS, "offset cap smaller than k");
    std::unordered_set<int64_t> chosen{cap};
    while ((int64_t)chosen.size() < k) chosen.insert(bounded(1, cap - 1));
    offs.assign(chosen.begin(), chosen.end());
    std::sort(offs.begin(), offs.end(), std::greater<>());
  }
  const int64_t a1 = offs.front();
  if (n <= a1) return fail(PIPEDP_E_INVALID_PARAMS, "n must exceed the largest offset");
  if (init_cap < a1) return fail(PIPEDP_E_INVALID_PARAMS, "init buffer holds %lld < a_1=%lld values",
                                 (long long)init_cap, (long long)a1);
  std::copy(offs.begin(), offs.end(), offsets_out);
  for (int64_t i = 0; i < a1; ++i) init_out[i] = bounded(0, (int64_t(1) << 20) - 1);
  if (a1_out) *a1_out = a1;
  return validate_sdp(offsets_out, k, a1, n);
}

// generate.cpp:49-60
int32_t pipedp_generate_mcm(int64_t n, uint64_t seed, int64_t dims_min, int64_t dims_max,
                            int64_t* dims_out) {
  if (n < 1) return fail(PIPEDP_E_INVALID_PARAMS, "n must be >= 1");
  if (dims_min < 1 || dims_min > dims_max) return fail(PIPEDP_E_INVALID_PARAMS, "bad dimension range");
  std::mt19937_64 rng(seed);
  for (int64_t i = 0; i <= n; ++i)
    dims_out[i] = dims_min + (int64_t)(rng() % (uint64_t)(dims_max - dims_min + 1));
  return validate_mcm(dims_out, n + 1);
}

// Batched generators (harness for the batch driver): instance i is exactly
// generate_sdp / generate_mcm with seed0 + i; every S-DP instance has a_1 = cap
// (or k when consecutive), so the outputs are dense SoA blocks.
int32_t pipedp_generate_sdp_batch(int64_t n, int64_t k, uint64_t seed0, int64_t count,
                                  int32_t consecutive, int64_t a1_cap, int64_t* offsets_out,
                                  int64_t* init_out, int64_t* a1_out) {
  if (count < 0 || k < 1) return fail(PIPEDP_E_INVALID_PARAMS, "bad batch shape");
  const int64_t a1 = consecutive ? k : (a1_cap > 0 ? a1_cap : 2 * k);
  if (a1_out) *a1_out = a1;
  const int nt = (int)std::max<int64_t>(1, std::min<int64_t>(count / 64 + 1, 32));
  std::vector<int32_t> rc(nt, PIPEDP_OK);
  std::vector<std::string> err(nt);
  auto work = [&](int t) {
    for (int64_t i = t; i < count; i += nt) {
      int64_t got = 0;
      const int r = pipedp_generate_sdp(n, k, 0, seed0 + (uint64_t)i, consecutive, a1_cap,
                                        offsets_out + i * k, init_out + i * a1, a1, &got);
      if (r != PIPEDP_OK) {
        rc[t] = r;
        err[t] = g_last_error;
        return;
      }
    }
  };
  std::vector<std::thread> th;
  for (int t = 1; t < nt; ++t) th.emplace_back(work, t);
  work(0);
  for (auto& x : th) x.join();
  for (int t = 0; t < nt; ++t)
    if (rc[t] != PIPEDP_OK) {
      g_last_error = err[t];
      return rc[t];
    }
  return PIPEDP_OK;
}

int32_t pipedp_generate_mcm_batch(int64_t n, uint64_t seed0, int64_t count, int64_t dims_min,
                                  int64_t dims_max, int64_t* dims_out) {
  if (count < 0) return fail(PIPEDP_E_INVALID_PARAMS, "bad batch shape");
  for (int64_t i = 0; i < count; ++i)
    TRY(pipedp_generate_mcm(n, seed0 + (uint64_t)i, dims_min, dims_max, dims_out + i * (n + 1)));
  return PIPEDP_OK;
}

// ------------------------------------------------------------- S-DP ---
int32_t pipedp_sdp_plan_create(int64_t batch, int64_t n, int64_t k, int64_t a1,
                               const int64_t* h_offsets, const int64_t* h_init, int32_t op,
                               int32_t device, pipedp_sdp_plan_t* plan_out) {
  if (!plan_out) return fail(PIPEDP_E_INVALID_PARAMS, "plan_out is NULL");
  *plan_out = nullptr;
  if (batch < 1) return fail(PIPEDP_E_INVALID_PARAMS, "batch must be >= 1");
  for (int64_t b = 0; b < batch; ++b) {
    TRY(validate_sdp(h_offsets + b * k, k, a1, n));
    if (h_offsets[b * k] != a1) return fail(PIPEDP_E_INIT_LENGTH_MISMATCH,
                                            "instance %lld has a_1=%lld, batch a_1=%lld",
                                            (long long)b, (long long)h_offsets[b * k], (long long)a1);
  }
  SdpDispatch d{};
  TRY(plan_sdp(batch, n, k, a1, h_offsets, h_init, op, &d));
  TRY(select_device(device));
  auto* P = new pipedp_sdp_plan{};
  CK(cudaGetDevice(&P->device));
  P->batch = batch;
  P->n = n;
  P->k = k;
  P->a1 = a1;
  P->d = d;
  cudaError_t e = cudaMalloc(&P->d_offsets, sizeof(int64_t) * batch * k);
  if (e == cudaSuccess)
    e = cudaMemcpy(P->d_offsets, h_offsets, sizeof(int64_t) * batch * k, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && d.remote) e = cudaMalloc(&P->d_remote, kRemoteBytes);
  if (e == cudaSuccess && d.remote) {
    std::vector<int32_t> obg((size_t)k);
    for (int64_t j = 0; j < k; ++j) obg[(size_t)j] = (int32_t)(h_offsets[j] * 8);
    e = cudaMalloc(&P->d_obg, sizeof(int32_t) * k);
    if (e == cudaSuccess) e = cudaMemcpy(P->d_obg, obg.data(), sizeof(int32_t) * k, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && d.warp_kernel && batch > 1 && (op == PIPEDP_OP_MIN || op == PIPEDP_OP_MAX)) {
    // group the instances that take the batch kernel's dominance form (offset 1,
    // a_1 <= 128) ahead of the others
    // modes as sdp_batch_warp decides them: 1 (offset 1), 2 (S* covers [2, 127]), 0
    std::vector<int> mode((size_t)batch, 0);
    for (int64_t b = 0; b < batch && a1 <= 128 && k >= 2; ++b) {
      const int64_t* o = h_offsets + b * k;
      bool has1 = false;
      for (int64_t j = 0; j < k; ++j) has1 = has1 || o[j] == 1;
      if (has1) {
        mode[(size_t)b] = 1;
        continue;
      }
      bool reach[128] = {true};
      bool all = true;
      for (int v = 1; v < 128; ++v) {
        for (int64_t j = 0; j < k && !reach[v]; ++j) reach[v] = o[j] <= v && reach[v - o[j]];
        if (v >= 2) all = all && reach[v];
      }
      if (all) mode[(size_t)b] = 2;
    }
    // the dominance kernel first (device-classified: g <= 32), then the rest by mode
    std::vector<pipedp_bdom::DomInfo> info;
    if (d.bits == 32 && a1 >= 64 && a1 <= 128 && env_int("PIPEDP_SDP_BDOM", 1) != 0) {
      e = cudaMalloc(&P->d_dinfo, sizeof(pipedp_bdom::DomInfo) * batch);
      if (e == cudaSuccess) e = pipedp_bdom::classify(batch, (int32_t)k, (int32_t)a1, P->d_offsets, P->d_dinfo, 0);
      if (e == cudaSuccess) {
        info.resize((size_t)batch);
        e = cudaMemcpy(info.data(), P->d_dinfo, sizeof(pipedp_bdom::DomInfo) * batch, cudaMemcpyDeviceToHost);
      }
    }
    std::vector<int32_t> perm;
    perm.reserve((size_t)batch);
    for (int64_t b = 0; b < (int64_t)info.size(); ++b)
      if (info[(size_t)b].g != 0) perm.push_back((int32_t)b);
    P->n_dom = (int64_t)perm.size();
    for (int want : {1, 2, 0})
      for (int64_t b = 0; b < batch; ++b)
        if (mode[(size_t)b] == want && (info.empty() || info[(size_t)b].g == 0)) perm.push_back((int32_t)b);
    e = cudaMalloc(&P->d_perm, sizeof(int32_t) * batch);
    if (e == cudaSuccess) e = cudaMemcpy(P->d_perm, perm.data(), sizeof(int32_t) * batch, cudaMemcpyHostToDevice);
  }
  if (e == cudaSuccess && d.chunked) {
    P->Lc = d.chunk_len;
    P->G = (n - a1 + P->Lc - 1) / P->Lc;
    P->n_i = a1 + P->Lc;
    // 64-bit words per row: rows padded to 2048 bits (whole 128-wide product
    // tiles and whole 64-word K stages)
    P->W = (int32_t)((a1 + 2047) / 2048 * 32);
    std::vector<int64_t> orep((size_t)(P->G * k)), irep((size_t)(P->G * a1));
    for (int64_t g = 0; g < P->G; ++g) {
      std::copy(h_offsets, h_offsets + k, orep.begin() + g * k);
      std::copy(h_init, h_init + a1, irep.begin() + g * a1);
    }
    const int rc = plan_sdp(P->G, P->n_i, k, a1, orep.data(), irep.data(), op, &P->dc);
    if (rc != PIPEDP_OK) {
      pipedp_sdp_plan_destroy(P);
      return rc;
    }
    // chunk CTAs: fewer, fuller far warps and one mid warp so two chunks share
    // an SM (the per-chunk pipeline is latency-bound; measured on the C2 shape:
    // 256 chunks 5.39 -> 4.67 ms)
    SdpDispatch& dc = P->dc;
    if (!dc.warp_kernel && !dc.remote && !dc.v2 && !dc.small && !dc.gfar) {
      int64_t jf = 0;
      // mid/far boundary 384 for wide states (C2: 5.81 -> 5.74 ms measured)
      const int amid = std::max(128, env_int("PIPEDP_CHUNK_AMID", a1 > 1024 ? 384 : kAMid)) & ~31;
      for (int64_t j = 0; j < k; ++j) jf += h_offsets[j] >= amid;
      dc.shape.a_mid = amid;
      dc.shape.mid_warps = std::max(1, env_int("PIPEDP_CHUNK_MID_WARPS", 1));
      dc.shape.far_warps = (int32_t)std::min<int64_t>(std::max(1, env_int("PIPEDP_CHUNK_FAR_WARPS", 8)),
                                                      std::max<int64_t>(1, (jf + 47) / 48));
      dc.threads = 32 * sdp_warps_for_roles(dc.shape.mid_warps + dc.shape.far_warps + 1);
    }
    const size_t mat = (size_t)64 * P->W * P->W;
    e = cudaMalloc(&P->d_bm, sizeof(unsigned long long) * 6 * mat);  // X, XT, Z, ZT, R, RT
    if (e == cudaSuccess) e = cudaMalloc(&P->d_q, sizeof(unsigned long long) * mat);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_E, sizeof(int64_t) * 2 * 64 * P->W + 512);  // + flags, barrier
    if (e == cudaSuccess) e = cudaMalloc(&P->d_cinit, sizeof(int64_t) * P->G * a1);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_offs_rep, sizeof(int64_t) * P->G * k);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_pad, sizeof(int64_t) * P->G * P->n_i);
    if (e == cudaSuccess)
      e = cudaMemcpy(P->d_offs_rep, orep.data(), sizeof(int64_t) * P->G * k, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && env_int("PIPEDP_SDP_RANK", 1) != 0) {
      auto* rp = new pipedp_rank::ChunkRankParams();
      if (pipedp_rank::chunk_rank_plan(h_offsets, P->d_offsets, (int)k, (int)a1, n, P->Lc, P->G,
                                       op == PIPEDP_OP_MAX ? 1 : 0, rp, &P->rank_threads, &P->rank_smem)) {
        P->rank = rp;
        e = cudaMalloc(&P->d_sorted, sizeof(int64_t) * a1);
      } else {
        delete rp;
      }
    }
  }
  if (e != cudaSuccess) {
    pipedp_sdp_plan_destroy(P);
    return cuda_fail(e, "sdp plan upload");
  }
  *plan_out = P;
  return PIPEDP_OK;
}

// fold the last recorded run's phase durations into the accumulators
static int phase_collect(pipedp_sdp_plan_t P) {
  if (!P->phase_pending) return PIPEDP_OK;
  CK(cudaEventSynchronize(P->ev_phase[3]));
  for (int i = 0; i < 3; ++i) {
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, P->ev_phase[i], P->ev_phase[i + 1]));
    P->phase_ms[i] += ms;
  }
  ++P->phase_runs;
  P->phase_pending = false;
  return PIPEDP_OK;
}

// Chunked mode (sdp_chunked.cuh): Q = M^Lc by boolean squarings, the chunk
// entry states by Q (.) state, then all chunks as one batch.
extern "C++" {
template <int OP>
static int32_t sdp_chunked_run(pipedp_sdp_plan_t P, const int64_t* d_init, int64_t* d_cells, cudaStream_t st,
                               int64_t split_at = 0, cudaEvent_t split_event = nullptr) {
  const int32_t W = P->W, a1 = (int32_t)P->a1;
  const size_t mat = (size_t)64 * W * W;
  if (P->timing) {
    TRY(phase_collect(P));  // the previous run's phases
    for (auto& e : P->ev_phase)
      if (!e) CK(cudaEventCreate(&e));
    CK(cudaEventRecord(P->ev_phase[0], st));
  }
  unsigned long long *X = P->d_bm, *XT = X + mat, *Z = XT + mat, *ZT = Z + mat;
  CK(cudaMemsetAsync(X, 0, sizeof(unsigned long long) * 2 * mat, st));
  bm_build<<<1, 1024, 0, st>>>(P->d_offsets, (int32_t)P->k, a1, W, X, XT);
  CK(cudaGetLastError());
  const size_t smem = sizeof(uint32_t) * (kBmR + kBmC) * (kBmK + 4);
  CK(cudaFuncSetAttribute(bm_mul, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const dim3 grid((unsigned)W, (unsigned)(W / 2));  // 128 x 64 output tiles
  auto x32 = [](const unsigned long long* p) { return reinterpret_cast<const uint32_t*>(p); };
  int* flags = reinterpret_cast<int*>(P->d_E + 2 * 64 * W);  // per-squaring changed flags
  CK(cudaMemsetAsync(flags, 0, sizeof(int) * 64, st));
  unsigned long long *R = ZT + mat, *RT = R + mat;
  // out = A B for the power M^t_new: rows >= t_new (t_new < a1) are shifts,
  // written directly; only the rows above them are multiplied
  // out = A B (and outT = out^T, written by the same kernels: the next
  // product's right operand)
  auto product = [&](const unsigned long long* A, const unsigned long long* BT, unsigned long long* out,
                     unsigned long long* outT, int64_t t_new, const int* prev, int* chg) {
    const int64_t rows = 64ll * W;
    const int64_t lim = t_new < a1 ? std::min<int64_t>(rows, (t_new + kBmR - 1) / kBmR * kBmR) : rows;
    bm_mul<<<dim3((unsigned)W, (unsigned)(lim / kBmR)), 256, smem, st>>>(x32(A), x32(BT), 2 * W, out, prev, chg,
                                                                          outT);
    if (lim < rows)
      bm_shift_rows<<<(unsigned)std::min<int64_t>(1024, ((rows - lim) * W + 255) / 256), 256, 0, st>>>(
          out, W, t_new, lim, a1, chg, outT);
  };
  int64_t ex = 1, er = 0;  // exponents of X and R
  auto square = [&](int i) {  // X <- X X (then its transpose); flags track idempotence
    product(X, XT, Z, ZT, 2 * ex, i ? flags + i - 1 : nullptr, flags + i);
    std::swap(X, Z);
    std::swap(XT, ZT);
    ex *= 2;
  };
  // Q = M^Lc by square-and-multiply over the bits of Lc (R accumulates)
  const int top = 63 - __builtin_clzll((unsigned long long)P->Lc);
  int nsq = 0;
  bool have_r = false;
  for (int i = 0; i <= top; ++i) {
    if ((P->Lc >> i) & 1) {
      if (!have_r) {
        CK(cudaMemcpyAsync(R, X, sizeof(unsigned long long) * 2 * mat, cudaMemcpyDeviceToDevice, st));  // R, RT
        have_r = true;
        er = ex;
      } else {  // R <- R X (powers of M commute)
        product(R, XT, Z, ZT, er + ex, nullptr, nullptr);
        std::swap(R, Z);
        std::swap(RT, ZT);
        er += ex;
      }
    }
    if (i < top) square(nsq++);
    CK(cudaGetLastError());
  }
  // from here X, XT hold Q
  std::swap(X, R);
  std::swap(XT, RT);
  CK(cudaMemsetAsync(flags + nsq, 0xFF, sizeof(int), st));  // Q's own squarings start fresh ("changed")
  int64_t* E[2] = {P->d_E, P->d_E + 64 * W};
  CK(cudaFuncSetAttribute(bm_matvec<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          (int)(sizeof(int64_t) * 64 * W)));
  if (P->timing) CK(cudaEventRecord(P->ev_phase[1], st));
  bm_state0<<<(a1 + 255) / 256, 256, 0, st>>>(d_init, a1, E[0], P->d_cinit);
  const int B = P->G >= 64 ? 16 : 1;  // two-level chain block
  if (env_int("PIPEDP_SDP_CHAIN_PERSISTENT", 1) != 0) {
    // Q_B = Q^B: log2(B) more squarings of the saved Q
    const unsigned long long* Q = X;
    unsigned long long* QB = X;
    if (B > 1) {
      CK(cudaMemcpyAsync(P->d_q, X, sizeof(unsigned long long) * mat, cudaMemcpyDeviceToDevice, st));
      Q = P->d_q;
      for (int b = 1, i = nsq + 1; b < B; b *= 2, ++i) {
        product(X, XT, Z, ZT, er * 2 * b, flags + i - 1, flags + i);
        CK(cudaGetLastError());
        std::swap(X, Z);
        std::swap(XT, ZT);
      }
      QB = X;
    }
    unsigned* bar = reinterpret_cast<unsigned*>(flags + 64);
    CK(cudaMemsetAsync(bar, 0, 2 * sizeof(unsigned), st));
    const size_t es = sizeof(int64_t) * 65 * W;  // E + per-word (x)
    CK(cudaFuncSetAttribute(bm_chain<OP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)es));
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, bm_chain<OP>, 1024, es));
    if (per_sm < 1) return fail(PIPEDP_ERR_UNSUPPORTED, "bm_chain does not fit an SM");
    const int nblk = sm_count();
    const unsigned long long* qb = QB;
    int32_t bb = B, w = W, a = a1;
    int64_t gg = P->G;
    int64_t* ci = P->d_cinit;
    void* args[] = {(void*)&Q, (void*)&qb, (void*)&bb, (void*)&w, (void*)&a, (void*)&gg, (void*)&ci, (void*)&bar};
    CK(cudaLaunchCooperativeKernel((const void*)bm_chain<OP>, dim3((unsigned)nblk), dim3(1024), args, es, st));
  } else {
    for (int64_t g = 1; g < P->G; ++g)
      bm_matvec<OP><<<(a1 + 7) / 8, 256, sizeof(int64_t) * 64 * W, st>>>(X, W, a1, E[(g - 1) & 1], E[g & 1],
                                                                         P->d_cinit + g * a1);
    CK(cudaGetLastError());
  }
  CK(cudaMemcpyAsync(d_cells, d_init, sizeof(int64_t) * a1, cudaMemcpyDeviceToDevice, st));
  if (P->timing) CK(cudaEventRecord(P->ev_phase[2], st));
  // chunks [0, gs) then [gs, G), each gathered into the instance's table; an
  // event after the first range lets the host copy it out while the second runs
  const int64_t gs = split_at > 0 && split_at < P->G ? split_at : P->G;
  if (P->rank) {  // rank-compressed chunk batch: chunks write the table directly
    CK(pipedp_rank::chunk_rank_sort(d_init, a1, P->d_sorted, st));
    P->rank->cinit = P->d_cinit;
    P->rank->sorted = P->d_sorted;
    P->rank->out = d_cells;
  }
  for (int64_t g0 = 0; g0 < P->G; g0 = gs == P->G ? P->G : (g0 == 0 ? gs : P->G)) {
    const int64_t g1 = g0 == 0 ? gs : P->G;
    if (P->rank) {
      P->rank->g0 = g0;
      P->rank->G = g1;
      CK(pipedp_rank::chunk_rank_launch(*P->rank, P->rank_threads, P->rank_smem, st));
      if (g0 == 0 && split_event) CK(cudaEventRecord(split_event, st));
      continue;
    }
    TRY(launch_sdp(P->dc, g1 - g0, P->d_offs_rep + g0 * P->k, P->d_cinit + g0 * a1, P->d_pad + g0 * P->n_i,
                   SdpRemote{}, st));
    const int64_t full = std::min(g1, P->G - 1) - g0;  // whole chunks in the range
    if (full > 0)
      CK(cudaMemcpy2DAsync(d_cells + a1 + g0 * P->Lc, sizeof(int64_t) * P->Lc, P->d_pad + g0 * P->n_i + a1,
                           sizeof(int64_t) * P->n_i, sizeof(int64_t) * P->Lc, (size_t)full,
                           cudaMemcpyDeviceToDevice, st));
    if (g1 == P->G) {  // the ragged last chunk
      const int64_t last = P->n - a1 - (P->G - 1) * P->Lc;
      CK(cudaMemcpyAsync(d_cells + a1 + (P->G - 1) * P->Lc, P->d_pad + (P->G - 1) * P->n_i + a1,
                         sizeof(int64_t) * last, cudaMemcpyDeviceToDevice, st));
    }
    if (g0 == 0 && split_event) CK(cudaEventRecord(split_event, st));
  }
  if (P->timing) {
    CK(cudaEventRecord(P->ev_phase[3], st));
    P->phase_pending = true;
  }
  return PIPEDP_OK;
}
}  // extern "C++"

// `armed` (optional) is recorded once the remote workspace is reset, before
// the launch: copies ordered after it may read the progress counters.
static int32_t sdp_execute(pipedp_sdp_plan_t P, const int64_t* d_init, int64_t* d_cells,
                           void* stream, cudaEvent_t armed) {
  if (P->d.chunked) {
    CK(cudaSetDevice(P->device));
    return P->d.op == PIPEDP_OP_MAX ? sdp_chunked_run<kMax>(P, d_init, d_cells, (cudaStream_t)stream)
                                    : sdp_chunked_run<kMin>(P, d_init, d_cells, (cudaStream_t)stream);
  }
  CK(cudaSetDevice(P->device));
  SdpRemote rm{};
  if (P->d.remote) {
    char* w = static_cast<char*>(P->d_remote);
    rm.part = w;
    rm.ready = reinterpret_cast<int*>(w + kRemSlots * 32 * sizeof(int64_t));
    rm.published = reinterpret_cast<unsigned long long*>(w + kRemSlots * 32 * sizeof(int64_t) + kRemSlots * sizeof(int));
    rm.obg = P->d_obg;
    CK(cudaMemsetAsync(P->d_remote, 0, kRemoteBytes, (cudaStream_t)stream));
    // producers read the preset prefix straight from the table before the
    // finisher CTA has necessarily run: stage it there in stream order
    CK(cudaMemcpyAsync(d_cells, d_init, sizeof(int64_t) * P->a1, cudaMemcpyDeviceToDevice,
                       (cudaStream_t)stream));
  }
  if (armed) CK(cudaEventRecord(armed, (cudaStream_t)stream));
  if (P->d_perm) {
    SdpDispatch dd = P->d;
    dd.shape.perm = P->d_perm + P->n_dom;
    if (P->n_dom == 0)
      return launch_sdp(dd, P->batch, P->d_offsets, d_init, d_cells, rm, (cudaStream_t)stream);
    const bool rest = P->n_dom < P->batch;
    if (rest) {  // the few sdp_batch_warp instances run beside the dominance kernel
      if (!P->side) {
        CK(cudaStreamCreateWithFlags(&P->side, cudaStreamNonBlocking));
        CK(cudaEventCreateWithFlags(&P->ev_fork, cudaEventDisableTiming));
        CK(cudaEventCreateWithFlags(&P->ev_join, cudaEventDisableTiming));
      }
      CK(cudaEventRecord(P->ev_fork, (cudaStream_t)stream));
      CK(cudaStreamWaitEvent(P->side, P->ev_fork, 0));
      TRY(launch_sdp(dd, P->batch - P->n_dom, P->d_offsets, d_init, d_cells, rm, P->side));
      CK(cudaEventRecord(P->ev_join, P->side));
    }
    CK(pipedp_bdom::launch(P->d.op == PIPEDP_OP_MAX ? 1 : 0, P->n_dom, P->d_perm, P->n, (int32_t)P->k,
                           (int32_t)P->a1, P->d_offsets, d_init, d_cells, P->d_dinfo, (cudaStream_t)stream));
    if (rest) CK(cudaStreamWaitEvent((cudaStream_t)stream, P->ev_join, 0));
    return PIPEDP_OK;
  }
  return launch_sdp(P->d, P->batch, P->d_offsets, d_init, d_cells, rm, (cudaStream_t)stream);
}

int32_t pipedp_sdp_plan_execute(pipedp_sdp_plan_t P, const int64_t* d_init, int64_t* d_cells,
                                void* stream) {
  if (!P) return fail(PIPEDP_E_INVALID_PARAMS, "null plan");
  return sdp_execute(P, d_init, d_cells, stream, nullptr);
}

// Remote-mode (multi-CTA) single-instance solves publish their finished
// prefix in `published` (batches of 32 cells past a1): copy the table out
// while the kernel is still producing its tail.
// The caller's `filled` flags (all ones on success, sdp.cpp:62-64): written by
// the copy pool while the kernels run, together with the output's prefault;
// whatever is left (paths without an overlap window) the caller writes after.
struct HostFill {
  uint8_t* p = nullptr;
  size_t n = 0;
};

static void host_prep(int64_t* cells_out, size_t bytes, HostFill* fill) {
  pipedp_host::parallel_prefault(cells_out, bytes);
  if (fill && fill->p) {
    pipedp_host::parallel_fill(fill->p, 1, fill->n);
    fill->p = nullptr;
  }
}

static int32_t sdp_execute_to_host(pipedp_sdp_plan_t P, pipedp_host::Workspace* W,
                                   const int64_t* d_init, int64_t* d_cells, int64_t* cells_out,
                                   const int64_t* h_init, HostFill* fill = nullptr) {
  const size_t bytes = sizeof(int64_t) * P->batch * P->n;
  if (P->rank && P->d.method == PIPEDP_SDP_PIPELINE && bytes >= kHostCopyBig && h_init &&
      env_int("PIPEDP_D2H_NARROW", 1) != 0) {
    // chunked min / max on ranks: the cells leave the device as 16-bit ranks
    // (2 B per cell) and become values on the host by a lookup into the
    // sorted init values -- the same multiset the device sorted, so the same
    // rank -> value map; the preset prefix is the caller's init
    void* d_rank = nullptr;
    CK(W->buffer(4, sizeof(uint16_t) * (size_t)(P->a1 + P->G * P->Lc) + 16, &d_rank));
    // progressive: every chunk publishes how far it is, and the finished
    // column band of all chunks leaves the device while they run
    const bool progressive = env_int("PIPEDP_D2H_PROGRESSIVE", 1) != 0;
    uint32_t epoch = 0;
    if (progressive) {
      CK(W->streaming_init());
      CK(W->progress_words((size_t)P->G));
      epoch = ++W->prog_epoch;
      P->rank->progress = W->prog_d;
      P->rank->epoch = epoch;
    }
    P->rank->out_rank = static_cast<uint16_t*>(d_rank);
    const int32_t rc = P->d.op == PIPEDP_OP_MAX ? sdp_chunked_run<kMax>(P, d_init, d_cells, W->stream)
                                                : sdp_chunked_run<kMin>(P, d_init, d_cells, W->stream);
    P->rank->out_rank = nullptr;
    P->rank->progress = nullptr;
    TRY(rc);
    if (progressive) CK(cudaEventRecord(W->done, W->stream));
    std::vector<int64_t> sorted(h_init, h_init + P->a1);
    std::sort(sorted.begin(), sorted.end());
    // first-touch the output while the kernels run (measured: faulting it in
    // from the conversion instead is 0.6 ms slower on C2)
    host_prep(cells_out, bytes, fill);
    memcpy(cells_out, h_init, sizeof(int64_t) * P->a1);
    if (progressive)
      CK(W->d2h_lookup16_chunks(cells_out, static_cast<const uint16_t*>(d_rank), P->a1, P->n, P->G, P->Lc,
                                sorted.data(), epoch, W->done));
    else
      CK(W->d2h_lookup16(cells_out + P->a1, static_cast<const uint16_t*>(d_rank) + P->a1,
                         (size_t)(P->n - P->a1), sorted.data()));
    return PIPEDP_OK;
  }
  // (chunked plans never run the remote pipeline: no progress counters)
  if (!(P->d.remote && !P->d.chunked && P->batch == 1 && P->d.method == PIPEDP_SDP_PIPELINE) ||
      bytes < (64u << 20) ||
      env_int("PIPEDP_STREAM_D2H", 1) == 0) {
    const int bits = P->d.chunked ? P->dc.bits : P->d.bits;
    const bool narrow = bits == 32 && P->d.method == PIPEDP_SDP_PIPELINE && bytes >= kHostCopyBig &&
                        env_int("PIPEDP_D2H_NARROW", 1) != 0;
    if (P->d.chunked && narrow && P->G > sm_count() && env_int("PIPEDP_CHUNK_OVERLAP", 0) != 0) {
      // chunks in two launches (one per SM, then the rest): the first range's
      // cells leave the device while the second range computes.  Off by
      // default (PIPEDP_CHUNK_OVERLAP=1): on C2 the split launch costs more
      // than the overlap saves (e2e 13.6 vs 12.2 ms measured)
      CK(W->streaming_init());
      CK(cudaSetDevice(P->device));
      const int64_t gs = sm_count();
      TRY(P->d.op == PIPEDP_OP_MAX ? sdp_chunked_run<kMax>(P, d_init, d_cells, W->stream, gs, W->armed)
                                   : sdp_chunked_run<kMin>(P, d_init, d_cells, W->stream, gs, W->armed));
      host_prep(cells_out, bytes, fill);  // overlaps the kernels
      // cells [0, cut) are final at `armed`; cut is even so both halves stay
      // 16-byte aligned for narrow_i64_i32's int4 loads
      const int64_t cut = (P->a1 + gs * P->Lc) & ~(int64_t)1;
      CK(cudaStreamWaitEvent(W->side, W->armed, 0));
      TRY(d2h_narrowed(W, 4, cells_out, d_cells, cut, W->side));
      TRY(d2h_narrowed(W, 5, cells_out + cut, d_cells + cut, P->n - cut, W->stream));
      return PIPEDP_OK;
    }
    TRY(sdp_execute(P, d_init, d_cells, W->stream, nullptr));
    if (bytes >= kHostCopyBig) host_prep(cells_out, bytes, fill);  // overlaps the kernel
    // 32-bit value class (min/max of int32 presets, normalised mod-add): every
    // table value fits int32 -- copy out half the bytes
    if (narrow) return d2h_narrowed(W, 4, cells_out, d_cells, P->batch * P->n);
    CK(W->d2h(cells_out, d_cells, bytes));
    return PIPEDP_OK;
  }
  CK(W->streaming_init());
  TRY(sdp_execute(P, d_init, d_cells, W->stream, W->armed));
  CK(cudaEventRecord(W->done, W->stream));
  CK(cudaStreamWaitEvent(W->side, W->armed, 0));
  const int writers = P->d.v2 ? P->d.s2.writers : 1;
  const char* published = static_cast<const char*>(P->d_remote) + kRemSlots * 32 * sizeof(int64_t) +
                          kRemSlots * sizeof(int);
  auto progress = [&](size_t* ready) -> cudaError_t {
    cudaError_t e = cudaMemcpyAsync(W->ctr, published, sizeof(unsigned long long) * writers,
                                    cudaMemcpyDeviceToHost, W->side);
    if (e == cudaSuccess) e = cudaStreamSynchronize(W->side);
    if (e != cudaSuccess) return e;
    unsigned long long m = W->ctr[0];  // every batch below min_w published[w] is in HBM
    for (int w = 1; w < writers; ++w) m = std::min(m, W->ctr[w]);
    *ready = (size_t)std::min<int64_t>(P->n, P->a1 + 32 * (int64_t)m) * sizeof(int64_t);
    return cudaSuccess;
  };
  CK(W->d2h_streamed(cells_out, d_cells, bytes, W->done, progress));
  return PIPEDP_OK;
}

int32_t pipedp_sdp_plan_describe(pipedp_sdp_plan_t P, char* name, size_t cap, int32_t* bits,
                                 int32_t* launches) {
  if (!P) return fail(PIPEDP_E_INVALID_PARAMS, "null plan");
  if (name && cap) {
    if (P->d.chunked)
      snprintf(name, cap, "sdp_chunked[L=%lld,G=%lld,%s]", (long long)P->Lc, (long long)P->G,
               P->rank ? "chunk_rank_kernel" : sdp_kernel_name(P->dc));
    else if (P->n_dom > 0)
      snprintf(name, cap, "sdp_batch_dom[%lld/%lld]%s", (long long)P->n_dom, (long long)P->batch,
               P->n_dom < P->batch ? "+sdp_batch_warp" : "");
    else snprintf(name, cap, "%s", sdp_kernel_name(P->d));
  }
  if (bits) *bits = P->d.chunked ? P->dc.bits : P->d.bits;
  // kernels (remote mode adds a memset + a prefix copy); chunked: build,
  // product + transpose per squaring, state 0, the persistent chain, the batch
  if (launches) {
    int32_t nl = 1;
    if (P->d.chunked) {  // the launches of sdp_chunked_run, counted by replaying its ladder
      const int top = 63 - __builtin_clzll((unsigned long long)P->Lc);
      auto prod = [&](int64_t t_new) { return 1 + (t_new < P->a1 ? 1 : 0); };  // mul (+ shift rows), transposes fused
      int64_t ex = 1, er = 0;
      nl = 1;  // build
      for (int i = 0; i <= top; ++i) {
        if ((P->Lc >> i) & 1) {
          if (er) nl += prod(er + ex);
          er += ex;
        }
        if (i < top) {
          nl += prod(2 * ex);
          ex *= 2;
        }
      }
      nl += 1;  // state 0
      if (P->G >= 64)
        for (int b = 1; b < 16; b *= 2) nl += prod(er * 2 * b);
      nl += 1 + 1;  // chain, chunk batch
      if (P->rank) nl += 1;  // rank sort
    } else if (P->n_dom > 0) {
      nl = 1 + (P->n_dom < P->batch ? 1 : 0);  // dominance kernel (+ sdp_batch_warp for the rest)
    }
    *launches = nl;
  }
  return PIPEDP_OK;
}

int32_t pipedp_sdp_plan_set_timing(pipedp_sdp_plan_t P, int32_t on) {
  if (!P) return fail(PIPEDP_E_INVALID_PARAMS, "null plan");
  P->timing = on != 0;
  P->phase_ms[0] = P->phase_ms[1] = P->phase_ms[2] = 0;
  P->phase_runs = 0;
  P->phase_pending = false;
  return PIPEDP_OK;
}

int32_t pipedp_sdp_plan_phase_ms(pipedp_sdp_plan_t P, double* out3, int64_t* runs) {
  if (!P) return fail(PIPEDP_E_INVALID_PARAMS, "null plan");
  TRY(phase_collect(P));
  for (int i = 0; i < 3; ++i) out3[i] = P->phase_ms[i];
  if (runs) *runs = P->phase_runs;
  return PIPEDP_OK;
}

int32_t pipedp_sdp_plan_set_method(pipedp_sdp_plan_t P, int32_t method) {
  if (!P) return fail(PIPEDP_E_INVALID_PARAMS, "null plan");
  if (method < PIPEDP_SDP_PIPELINE || method > PIPEDP_SDP_NAIVE)
    return fail(PIPEDP_E_INVALID_PARAMS, "unknown S-DP method %d", method);
  if (method != PIPEDP_SDP_PIPELINE && P->batch != 1)
    return fail(PIPEDP_E_INVALID_PARAMS, "the paper's comparison methods solve one instance at a time");
  // int64 kernels; a non-associative instance (mixed-sign saturating-add)
  // keeps the strict-order pipeline, which is what the reference computes
  if (method != PIPEDP_SDP_PIPELINE && P->d.bits == 32) {
    P->d.bits = 64;
    P->d.vals32 = true;  // (the tournament keeps its shared-memory ring in 4-byte words)
  }
  P->d.method = method;
  if (method != PIPEDP_SDP_PIPELINE) P->d.chunked = false;  // the paper's methods run the instance as is
  return PIPEDP_OK;
}

int32_t pipedp_sdp_plan_destroy(pipedp_sdp_plan_t P) {
  if (!P) return PIPEDP_OK;
  cudaSetDevice(P->device);
  cudaFree(P->d_offsets);
  cudaFree(P->d_remote);
  cudaFree(P->d_obg);
  cudaFree(P->d_bm);
  cudaFree(P->d_q);
  cudaFree(P->d_perm);
  cudaFree(P->d_E);
  cudaFree(P->d_cinit);
  cudaFree(P->d_offs_rep);
  cudaFree(P->d_pad);
  cudaFree(P->d_sorted);
  cudaFree(P->d_dinfo);
  if (P->side) cudaStreamDestroy(P->side);
  for (auto e : P->ev_phase)
    if (e) cudaEventDestroy(e);
  if (P->ev_fork) cudaEventDestroy(P->ev_fork);
  if (P->ev_join) cudaEventDestroy(P->ev_join);
  delete P->rank;
  delete P;
  return PIPEDP_OK;
}

// Host-buffer solves: cached device buffers + staged, double-buffered copies
// (host_io.hpp); the tables themselves come only from the kernels.
static int32_t sdp_solve_host(int64_t batch, int64_t n, int64_t k, int64_t a1,
                              const int64_t* offsets, const int64_t* init, int32_t op,
                              int64_t* cells_out, int32_t device, HostFill* fill = nullptr) {
  // The last plan of this thread is kept (as for MCM): a caller re-solving an
  // instance with the same offsets (the reference's bench loops) skips the
  // planning uploads and allocations.  The dispatch is re-planned every call
  // (it depends on the init values' class and the environment) and must match.
  struct Cached {
    pipedp_sdp_plan_t plan = nullptr;
    std::vector<int64_t> offsets;
    int32_t op = -1;
    ~Cached() { pipedp_sdp_plan_destroy(plan); }
  };
  thread_local Cached cache;
  pipedp_sdp_plan_t P = nullptr;
  {
    TRY(select_device(device));
    int dev = 0;
    CK(cudaGetDevice(&dev));
    pipedp_sdp_plan_t C = cache.plan;
    if (C && C->device == dev && C->batch == batch && C->n == n && C->k == k && C->a1 == a1 && cache.op == op &&
        std::equal(cache.offsets.begin(), cache.offsets.end(), offsets) && cache.offsets.size() == (size_t)(batch * k)) {
      SdpDispatch d{};  // value-initialised like the cached one, so padding compares equal
      TRY(plan_sdp(batch, n, k, a1, offsets, init, op, &d));
      if (memcmp(&d, &C->d, sizeof d) == 0) P = C;
    }
  }
  if (!P) {
    pipedp_sdp_plan_destroy(cache.plan);
    cache.plan = nullptr;
    TRY(pipedp_sdp_plan_create(batch, n, k, a1, offsets, init, op, device, &P));
    cache.plan = P;
    cache.offsets.assign(offsets, offsets + batch * k);
    cache.op = op;
  } else {
    CK(cudaSetDevice(P->device));
  }
  pipedp_host::Workspace* W = nullptr;
  CK(pipedp_host::workspace(P->device, &W));
  void *d_init = nullptr, *d_cells = nullptr;
  CK(W->buffer(0, sizeof(int64_t) * batch * a1, &d_init));
  CK(W->buffer(1, sizeof(int64_t) * batch * n, &d_cells));
  CK(W->h2d(d_init, init, sizeof(int64_t) * batch * a1));
  return sdp_execute_to_host(P, W, (const int64_t*)d_init, (int64_t*)d_cells, cells_out, init, fill);
}

int32_t pipedp_sdp_solve(const int64_t* offsets, int64_t k, const int64_t* init,
                         int64_t init_len, int64_t n, int32_t op, int64_t* cells_out,
                         uint8_t* filled_out) {
  TRY(validate_sdp(offsets, k, init_len, n));
  HostFill fill{filled_out, (size_t)n};
  TRY(sdp_solve_host(1, n, k, init_len, offsets, init, op, cells_out, -1, &fill));
  if (fill.p) memset(fill.p, 1, fill.n);
  return PIPEDP_OK;
}

int32_t pipedp_sdp_solve_method(const int64_t* offsets, int64_t k, const int64_t* init,
                                int64_t init_len, int64_t n, int32_t op, int32_t method,
                                int64_t* cells_out, uint8_t* filled_out) {
  TRY(validate_sdp(offsets, k, init_len, n));
  pipedp_sdp_plan_t P = nullptr;
  TRY(pipedp_sdp_plan_create(1, n, k, init_len, offsets, init, op, -1, &P));
  struct Guard {
    pipedp_sdp_plan_t p;
    ~Guard() { pipedp_sdp_plan_destroy(p); }
  } guard{P};
  TRY(pipedp_sdp_plan_set_method(P, method));
  pipedp_host::Workspace* W = nullptr;
  CK(pipedp_host::workspace(P->device, &W));
  void *d_init = nullptr, *d_cells = nullptr;
  CK(W->buffer(0, sizeof(int64_t) * init_len, &d_init));
  CK(W->buffer(1, sizeof(int64_t) * n, &d_cells));
  CK(W->h2d(d_init, init, sizeof(int64_t) * init_len));
  TRY(pipedp_sdp_plan_execute(P, (const int64_t*)d_init, (int64_t*)d_cells, W->stream));
  CK(W->d2h(cells_out, d_cells, sizeof(int64_t) * n));
  if (filled_out) memset(filled_out, 1, (size_t)n);
  return PIPEDP_OK;
}

int32_t pipedp_sdp_solve_batch(int64_t batch, int64_t n, int64_t k, int64_t a1,
                               const int64_t* offsets, const int64_t* init, int32_t op,
                               int64_t* cells_out, int32_t device) {
  return sdp_solve_host(batch, n, k, a1, offsets, init, op, cells_out, device);
}

// -------------------------------------------------------------- MCM ---
int32_t pipedp_mcm_plan_create(int64_t batch, int64_t n, const int64_t* h_dims, int32_t kernel,
                               int32_t device, pipedp_mcm_plan_t* plan_out) {
  if (!plan_out) return fail(PIPEDP_E_INVALID_PARAMS, "plan_out is NULL");
  *plan_out = nullptr;
  if (batch < 1) return fail(PIPEDP_E_INVALID_PARAMS, "batch must be >= 1");
  if (n < 1) return fail(PIPEDP_E_INVALID_PARAMS, "dimension vector needs at least two entries");
  for (int64_t b = 0; b < batch; ++b) TRY(validate_mcm(h_dims + b * (n + 1), n + 1));
  McmDispatch d{};
  TRY(plan_mcm(batch, n, h_dims, kernel, &d));
  TRY(select_device(device));
  auto* P = new pipedp_mcm_plan{};
  P->batch = batch;
  P->n = n;
  {
    int64_t maxd = 0;
    for (int64_t i = 0; i < batch * (n + 1); ++i) maxd = std::max(maxd, h_dims[i]);
    P->maxd3 = maxd * maxd * maxd;  // dims validated <= 1e6: no overflow
  }
  P->cc = n * (n + 1) / 2;
  P->d = d;
  auto cleanup = [&](cudaError_t e, const char* what) {
    pipedp_mcm_plan_destroy(P);
    return cuda_fail(e, what);
  };
  cudaError_t e = cudaGetDevice(&P->device);
  std::vector<int32_t> p32((size_t)(batch * (n + 1)));
  for (size_t i = 0; i < p32.size(); ++i) p32[i] = (int32_t)h_dims[i];
  if (e == cudaSuccess) e = cudaMalloc(&P->d_p, sizeof(int32_t) * p32.size());
  if (e == cudaSuccess) e = cudaMemcpy(P->d_p, p32.data(), sizeof(int32_t) * p32.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&P->d_dims, sizeof(int64_t) * p32.size());
  if (e == cudaSuccess) e = cudaMemcpy(P->d_dims, h_dims, sizeof(int64_t) * p32.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&P->d_overflow, 4 * sizeof(int));  // + tournament grid barrier
  if (e == cudaSuccess) e = cudaMallocHost(&P->h_overflow, sizeof(int));
  if (e == cudaSuccess && d.kernel == PIPEDP_MCM_TILED) {
    const int64_t T = d.tile, TC = T * T;
    const int64_t N = (n + T - 1) / T, ntiles = N * (N + 1) / 2;
    P->N = (int32_t)N;
    std::vector<int32_t> pp((size_t)(N * T + 2), 0);
    for (int64_t i = 0; i <= n; ++i) pp[(size_t)i] = (int32_t)h_dims[i];
    const std::vector<unsigned long long> tasks = mcm_tiled_tasks((int)N);
    P->ntasks = (int64_t)tasks.size();
    e = cudaMalloc(&P->d_pp, sizeof(int32_t) * pp.size());
    if (e == cudaSuccess) e = cudaMemcpy(P->d_pp, pp.data(), sizeof(int32_t) * pp.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_tiles, sizeof(uint32_t) * ntiles * TC);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_keys, sizeof(unsigned long long) * ntiles * TC);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_tile_flags, sizeof(int) * 2 * ntiles);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_tasks, sizeof(unsigned long long) * tasks.size());
    if (e == cudaSuccess)
      e = cudaMemcpy(P->d_tasks, tasks.data(), sizeof(unsigned long long) * tasks.size(), cudaMemcpyHostToDevice);
    const void* kern = T == 32 ? (const void*)t32::mcm_tiled_kernel : (const void*)t64::mcm_tiled_kernel;
    const size_t ksmem = T == 32 ? t32::kTiledSmemBytes : t64::kTiledSmemBytes;
    if (e == cudaSuccess) e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ksmem);
    int per_sm = 0;
    if (e == cudaSuccess) e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTiledThreads, ksmem);
    // persistent grid: every CTA resident (tasks wait on earlier tasks only)
    P->tiled_grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)std::max(per_sm, 1) * sm_count(), P->ntasks));
    if (e == cudaSuccess && per_sm < 1) e = cudaErrorInvalidConfiguration;
  }
  // the wavefront resources also back the tiled kernel's exact int64 rerun
  const bool smem_may_fall_back = d.kernel == PIPEDP_MCM_SMEM && d.bits == 32 && d.smem64 > 227 * 1024;
  if (e == cudaSuccess &&
      (d.kernel == PIPEDP_MCM_WAVEFRONT || d.kernel == PIPEDP_MCM_TILED || smem_may_fall_back)) {
    std::vector<int64_t> base((size_t)n + 1, 0);
    int64_t total = 0;
    for (int64_t D = 1; D < n; ++D) {
      base[(size_t)D] = total;
      const int cpw = 32 / mcm_wave_group(D);
      total += (n - D + cpw - 1) / cpw;
    }
    P->total_chunks = total;
    e = cudaMalloc(&P->d_chunk_base, sizeof(int64_t) * (n + 1));
    if (e == cudaSuccess)
      e = cudaMemcpy(P->d_chunk_base, base.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_done, sizeof(int) * std::max<int64_t>(total, 1));
    if (e == cudaSuccess) e = cudaMalloc(&P->d_next, sizeof(unsigned long long));
    if (e == cudaSuccess) e = cudaMalloc(&P->d_v32, sizeof(uint32_t) * (P->cc + 1));
  }
  if (e != cudaSuccess) return cleanup(e, "mcm plan setup");
  *plan_out = P;
  return PIPEDP_OK;
}

int32_t pipedp_mcm_plan_execute(pipedp_mcm_plan_t P, int64_t* d_cells, int64_t* d_split, void* stream) {
  if (!P) return fail(PIPEDP_E_INVALID_PARAMS, "null plan");
  CK(cudaSetDevice(P->device));
  return mcm_execute(P, d_cells, d_split, (cudaStream_t)stream);
}

int32_t pipedp_mcm_plan_describe(pipedp_mcm_plan_t P, char* name, size_t cap, int32_t* bits,
                                 int32_t* launches) {
  if (!P) return fail(PIPEDP_E_INVALID_PARAMS, "null plan");
  TRY(mcm_resolve(P));  // an asynchronous execute: read its overflow bits
  const bool square = mcm_square_bytes(P->n, (P->last_bits ? P->last_bits : P->d.bits) / 8) <= kSmemBudget &&
                      env_int("PIPEDP_MCM_SQUARE", 1) != 0;
  const int lb = P->last_bits ? P->last_bits : P->d.bits;
  // the kernel mcm_smem_launch picks (packed_now: this plan's last execute)
  const bool bwarp = lb == 32 && P->packed_now && P->n <= pipedp_mcmb::kMaxN && env_int("PIPEDP_MCM_BATCH_WARP", 1) != 0;
  const char* nm = P->d.kernel == PIPEDP_MCM_SMEM         ? (bwarp ? "mcm_batch_warp" : square ? "mcm_smem_square" : "mcm_smem_cta")
                   : P->d.kernel == PIPEDP_MCM_TOURNAMENT ? "mcm_tournament_diag"
                   : (P->d.kernel == PIPEDP_MCM_TILED && P->last_bits != 64)
                       ? (P->d.tile == 32 ? "mcm_tiled_kernel<32>" : "mcm_tiled_kernel<64>")
                                                          : "mcm_wavefront";
  if (name && cap) snprintf(name, cap, "%s", nm);
  if (bits) *bits = P->last_bits ? P->last_bits : P->d.bits;
  if (launches) *launches = P->launches;
  return PIPEDP_OK;
}

int32_t pipedp_mcm_plan_destroy(pipedp_mcm_plan_t P) {
  if (!P) return PIPEDP_OK;
  cudaSetDevice(P->device);
  cudaFree(P->d_p);
  cudaFree(P->d_dims);
  cudaFree(P->d_v32);
  cudaFree(P->d_chunk_base);
  cudaFree(P->d_done);
  cudaFree(P->d_next);
  cudaFree(P->d_overflow);
  cudaFree(P->d_pp);
  cudaFree(P->d_tiles);
  cudaFree(P->d_keys);
  cudaFree(P->d_tile_flags);
  cudaFree(P->d_tasks);
  if (P->h_overflow) cudaFreeHost(P->h_overflow);
  if (P->ev_done) cudaEventDestroy(P->ev_done);
  delete P;
  return PIPEDP_OK;
}

// Re-upload a new batch of dims into an existing plan of the same shape and
// dispatch (the scratch tables are reused; only the dims-derived arrays change).
static int mcm_plan_reload(pipedp_mcm_plan_t P, const int64_t* h_dims, const McmDispatch& d) {
  const int64_t cnt = P->batch * (P->n + 1);
  {
    int64_t maxd = 0;
    for (int64_t i = 0; i < cnt; ++i) maxd = std::max(maxd, h_dims[i]);
    P->maxd3 = maxd * maxd * maxd;
  }
  std::vector<int32_t> p32((size_t)cnt);
  for (int64_t i = 0; i < cnt; ++i) p32[(size_t)i] = (int32_t)h_dims[i];
  CK(cudaSetDevice(P->device));
  CK(cudaMemcpy(P->d_p, p32.data(), sizeof(int32_t) * cnt, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(P->d_dims, h_dims, sizeof(int64_t) * cnt, cudaMemcpyHostToDevice));
  if (P->d_pp) {  // tiled: first n+1 entries (the zero padding is unchanged)
    CK(cudaMemcpy(P->d_pp, p32.data(), sizeof(int32_t) * (P->n + 1), cudaMemcpyHostToDevice));
  }
  P->d = d;
  P->launches = 0;
  P->last_bits = 0;
  return PIPEDP_OK;
}

static int32_t mcm_solve_host(int64_t batch, int64_t n, const int64_t* dims, int32_t kernel,
                              int64_t* cells_out, int64_t* split_out, int32_t device, HostFill* fill = nullptr) {
  // The last plan of this thread is kept: a caller solving instance after
  // instance of one shape (the reference's bench/verify loops) reuses its
  // device tables instead of reallocating hundreds of MiB per call.
  struct Cached {
    pipedp_mcm_plan_t plan = nullptr;
    int64_t batch = 0, n = 0;
    int32_t kernel = -1, device = -2;
    ~Cached() { pipedp_mcm_plan_destroy(plan); }
  };
  thread_local Cached cache;
  for (int64_t b = 0; b < batch; ++b) TRY(validate_mcm(dims + b * (n + 1), n + 1));
  McmDispatch d{};
  TRY(plan_mcm(batch, n, dims, kernel, &d));
  TRY(select_device(device));  // NoDevice without a GPU: there is no CPU path
  int dev = device;
  if (dev < 0) CK(cudaGetDevice(&dev));
  pipedp_mcm_plan_t P = nullptr;
  if (cache.plan && cache.batch == batch && cache.n == n && cache.kernel == kernel && cache.device == dev &&
      cache.plan->d.tile == d.tile && cache.plan->d.bits == d.bits) {
    P = cache.plan;
    TRY(mcm_plan_reload(P, dims, d));
  } else {
    pipedp_mcm_plan_destroy(cache.plan);
    cache.plan = nullptr;
    TRY(pipedp_mcm_plan_create(batch, n, dims, kernel, device, &P));
    cache.plan = P;
    cache.batch = batch;
    cache.n = n;
    cache.kernel = kernel;
    cache.device = dev;
  }
  const int64_t size = batch * (n * (n + 1) / 2 + 1);
  pipedp_host::Workspace* W = nullptr;
  CK(pipedp_host::workspace(P->device, &W));
  void *d_cells = nullptr, *d_split = nullptr;
  CK(W->buffer(1, sizeof(int64_t) * size, &d_cells));
  CK(W->buffer(2, sizeof(int64_t) * size, &d_split));
  // first-touch the host outputs while the kernels run (execute may wait on
  // the device for the overflow check)
  std::thread touch;
  if (sizeof(int64_t) * size >= kHostCopyBig)
    touch = std::thread([&] {
      pipedp_host::parallel_prefault(cells_out, sizeof(int64_t) * size);
      if (split_out) pipedp_host::parallel_prefault(split_out, sizeof(int64_t) * size);
      if (fill && fill->p) {
        pipedp_host::parallel_fill(fill->p, 1, fill->n);
        fill->p = nullptr;
      }
    });
  int32_t rc = pipedp_mcm_plan_execute(P, (int64_t*)d_cells, (int64_t*)d_split, W->stream);
  if (rc == PIPEDP_OK) rc = mcm_resolve(P);  // which attempt's table stands (its value width)
  if (touch.joinable()) touch.join();
  TRY(rc);
  // 32-bit run without the overflow flag: every cell < 2^30; split indices
  // always fit int32 -- copy out half the bytes
  const bool narrow = sizeof(int64_t) * size >= kHostCopyBig && env_int("PIPEDP_D2H_NARROW", 1) != 0;
  if (narrow && P->last_bits == 32) TRY(d2h_narrowed(W, 4, cells_out, (const int64_t*)d_cells, size));
  else CK(W->d2h(cells_out, d_cells, sizeof(int64_t) * size));
  if (split_out && narrow) {
    TRY(d2h_narrowed(W, 5, split_out, (const int64_t*)d_split, size));
    split_out = nullptr;  // done
  }
  if (split_out) CK(W->d2h(split_out, d_split, sizeof(int64_t) * size));
  return PIPEDP_OK;
}

int32_t pipedp_mcm_solve(const int64_t* dims, int64_t dims_len, int32_t kernel,
                         int64_t* cells_out, uint8_t* filled_out, int64_t* split_out) {
  TRY(validate_mcm(dims, dims_len));
  const int64_t n = dims_len - 1;
  HostFill fill{filled_out, (size_t)(n * (n + 1) / 2 + 1)};
  TRY(mcm_solve_host(1, n, dims, kernel, cells_out, split_out, -1, &fill));
  if (fill.p) memset(fill.p, 1, fill.n);
  return PIPEDP_OK;
}

int32_t pipedp_mcm_solve_batch(int64_t batch, int64_t n, const int64_t* dims, int64_t* cells_out,
                               int64_t* split_out, int32_t device) {
  return mcm_solve_host(batch, n, dims, PIPEDP_MCM_AUTO, cells_out, split_out, device);
}

int32_t pipedp_mcm_bruteforce(const int64_t* dims, int64_t dims_len, int64_t* out) {
  TRY(validate_mcm(dims, dims_len));
  const int64_t n = dims_len - 1;
  if (n > 12)
    return fail(PIPEDP_E_TOO_LARGE_FOR_BRUTE, "n=%lld exceeds the enumeration limit of 12", (long long)n);
  TRY(select_device(-1));
  Scope sc;
  TRY(sc.init());
  int64_t *d_p = nullptr, *d_out = nullptr;
  TRY(sc.alloc(&d_p, n + 1));
  TRY(sc.alloc(&d_out, 1));
  CK(cudaMemcpyAsync(d_p, dims, sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, sc.stream));
  mcm_bruteforce_kernel<<<1, 32, 0, sc.stream>>>(d_p, (int)n, d_out);
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(out, d_out, sizeof(int64_t), cudaMemcpyDeviceToHost, sc.stream));
  CK(cudaStreamSynchronize(sc.stream));
  return PIPEDP_OK;
}

// ------------------------------------------------------------ utilities ---
}  // extern "C"

namespace {
__global__ void fnv_digest_kernel(const int64_t* __restrict__ t, int64_t count, int64_t ntables,
                                  uint64_t* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= ntables) return;
  const int64_t* c = t + i * count;
  uint64_t h = 14695981039346656037ull;
  auto mix = [&](uint64_t v) {
#pragma unroll
    for (int b = 0; b < 8; ++b) {
      h ^= (v >> (8 * b)) & 0xffu;
      h *= 1099511628211ull;
    }
  };
  mix((uint64_t)count);
  for (int64_t j = 0; j < count; ++j) mix((uint64_t)__ldg(c + j));
  out[i] = h;
}
}  // namespace

extern "C" {

int32_t pipedp_digest_device(const int64_t* d_tables, int64_t count, int64_t ntables,
                             uint64_t* d_digests, void* stream) {
  if (ntables <= 0) return PIPEDP_OK;
  fnv_digest_kernel<<<(unsigned)((ntables + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
      d_tables, count, ntables, d_digests);
  CK(cudaGetLastError());
  return PIPEDP_OK;
}

int32_t pipedp_chain_fold_cycles(uint32_t hi, uint32_t m32, int32_t mode, double* cycles_out) {
  TRY(select_device(-1));
  Scope sc;
  TRY(sc.init());
  long long* d_cyc = nullptr;
  int32_t* d_sink = nullptr;
  TRY(sc.alloc(&d_cyc, 1));
  TRY(sc.alloc(&d_sink, 32));
  for (int rep = 0; rep < 2; ++rep)
    sdp_chain_fold_probe<kMin, int32_t><<<1, 32, 0, sc.stream>>>(1 << 14, hi, m32, mode, d_cyc, d_sink);
  CK(cudaGetLastError());
  long long c = 0;
  CK(cudaMemcpyAsync(&c, d_cyc, sizeof c, cudaMemcpyDeviceToHost, sc.stream));
  CK(cudaStreamSynchronize(sc.stream));
  *cycles_out = (double)c;
  return PIPEDP_OK;
}

int32_t pipedp_profile_read(uint64_t* out, int32_t count, int32_t reset) {
#ifdef PIPEDP_PROFILE
  unsigned long long h[128], hc[128];
  CK(cudaMemcpyFromSymbol(h, pipedp_dev::g_prof, sizeof h));
  CK(pipedp_cluster::profile_take(hc, reset != 0));  // the cluster TU's counters
  for (int i = 0; i < 128; ++i) h[i] += hc[i];
  for (int i = 0; i < count && i < 128; ++i) out[i] = h[i];
  if (reset) {
    memset(h, 0, sizeof h);
    CK(cudaMemcpyToSymbol(pipedp_dev::g_prof, h, sizeof h));
  }
  return PIPEDP_OK;
#else
  for (int i = 0; i < count; ++i) out[i] = 0;
  (void)reset;
  return fail(PIPEDP_ERR_UNSUPPORTED, "library built without -DPIPEDP_PROFILE");
#endif
}

int32_t pipedp_chain_step_ns(int32_t op, int32_t value_bits, int32_t device, double* ns_out,
                             double* mhz_out) {
  TRY(select_device(device));
  Scope sc;
  TRY(sc.init());
  long long* d_cyc = nullptr;
  int64_t* d_sink = nullptr;
  TRY(sc.alloc(&d_cyc, 1));
  TRY(sc.alloc(&d_sink, 32));
  const int64_t batches = 1 << 16;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&]() -> int {
    CK(cudaEventRecord(e0, sc.stream));
    switch (op * 100 + value_bits) {
      case 32: sdp_chain_step_probe<kMin, int32_t><<<1, 32, 0, sc.stream>>>(batches, 1, d_cyc, (int32_t*)d_sink); break;
      case 64: sdp_chain_step_probe<kMin, int64_t><<<1, 32, 0, sc.stream>>>(batches, 1, d_cyc, d_sink); break;
      case 132: sdp_chain_step_probe<kMax, int32_t><<<1, 32, 0, sc.stream>>>(batches, 1, d_cyc, (int32_t*)d_sink); break;
      case 164: sdp_chain_step_probe<kMax, int64_t><<<1, 32, 0, sc.stream>>>(batches, 1, d_cyc, d_sink); break;
      case 264: sdp_chain_step_probe<kSatAdd, int64_t><<<1, 32, 0, sc.stream>>>(batches, 1, d_cyc, d_sink); break;
      case 332: sdp_chain_step_probe<kModAdd, int32_t><<<1, 32, 0, sc.stream>>>(batches, 1, d_cyc, (int32_t*)d_sink); break;
      case 364: sdp_chain_step_probe<kModAdd, int64_t><<<1, 32, 0, sc.stream>>>(batches, 1, d_cyc, d_sink); break;
      default: return fail(PIPEDP_E_INVALID_PARAMS, "no chain probe for op %d at %d bits", op, value_bits);
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, sc.stream));
    CK(cudaEventSynchronize(e1));
    return PIPEDP_OK;
  };
  TRY(run());  // warm-up
  TRY(run());
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  long long cyc = 0;
  CK(cudaMemcpy(&cyc, d_cyc, sizeof cyc, cudaMemcpyDeviceToHost));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double steps = (double)batches * 32.0;
  if (ns_out) *ns_out = ms * 1e6 / steps;
  if (mhz_out) *mhz_out = (double)cyc / (ms * 1e3);
  return PIPEDP_OK;
}

int32_t pipedp_op_latency_ns(int32_t op, int32_t value_bits, int32_t device, double* ns_out,
                             double* cycles_out) {
  TRY(select_device(device));
  Scope sc;
  TRY(sc.init());
  long long* d_cyc = nullptr;
  int64_t* d_vals = nullptr;
  int64_t* d_sink = nullptr;
  TRY(sc.alloc(&d_cyc, 1));
  TRY(sc.alloc(&d_vals, 16));
  TRY(sc.alloc(&d_sink, 1));
  // operands that keep every op "live": small positive values (no saturation,
  // mod-add stays in range, min/max alternate)
  const int64_t h64[9] = {17, 3, 29, 5, 11, 23, 7, 13, 19};
  const int32_t h32[9] = {17, 3, 29, 5, 11, 23, 7, 13, 19};
  if (value_bits == 32) CK(cudaMemcpy(d_vals, h32, sizeof h32, cudaMemcpyHostToDevice));
  else CK(cudaMemcpy(d_vals, h64, sizeof h64, cudaMemcpyHostToDevice));
  const int64_t iters = 1 << 16;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  auto run = [&]() -> int {
    CK(cudaEventRecord(e0, sc.stream));
    int32_t* v32 = reinterpret_cast<int32_t*>(d_vals);
    int32_t* s32 = reinterpret_cast<int32_t*>(d_sink);
    switch (op * 100 + value_bits) {
      case 32: op_latency_probe<kMin, int32_t><<<1, 1, 0, sc.stream>>>(iters, v32, d_cyc, s32); break;
      case 64: op_latency_probe<kMin, int64_t><<<1, 1, 0, sc.stream>>>(iters, d_vals, d_cyc, d_sink); break;
      case 132: op_latency_probe<kMax, int32_t><<<1, 1, 0, sc.stream>>>(iters, v32, d_cyc, s32); break;
      case 164: op_latency_probe<kMax, int64_t><<<1, 1, 0, sc.stream>>>(iters, d_vals, d_cyc, d_sink); break;
      case 264: op_latency_probe<kSatAdd, int64_t><<<1, 1, 0, sc.stream>>>(iters, d_vals, d_cyc, d_sink); break;
      case 332: op_latency_probe<kModAdd, int32_t><<<1, 1, 0, sc.stream>>>(iters, v32, d_cyc, s32); break;
      case 364: op_latency_probe<kModAdd, int64_t><<<1, 1, 0, sc.stream>>>(iters, d_vals, d_cyc, d_sink); break;
      default: return fail(PIPEDP_E_INVALID_PARAMS, "no latency probe for op %d at %d bits", op, value_bits);
    }
    CK(cudaGetLastError());
    CK(cudaEventRecord(e1, sc.stream));
    CK(cudaEventSynchronize(e1));
    return PIPEDP_OK;
  };
  TRY(run());
  TRY(run());
  float ms = 0.f;
  CK(cudaEventElapsedTime(&ms, e0, e1));
  long long cyc = 0;
  CK(cudaMemcpy(&cyc, d_cyc, sizeof cyc, cudaMemcpyDeviceToHost));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double ops = (double)iters * 8.0;
  if (ns_out) *ns_out = ms * 1e6 / ops;
  if (cycles_out) *cycles_out = (double)cyc / ops;
  return PIPEDP_OK;
}

}  // extern "C"
