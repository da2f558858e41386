// evaluator.cu — K6/K7: DreamShard's cost network and policy network,
// batched over candidate placements on one GPU (fp32 CUDA cores; the MLPs
// are 21-128-32 / 32-64-1 / 3-64-32 / 64-1, far too small for tensor cores).
//
//   sp_eval_batch    EstimatedCostProvider::overall + cost_features for many
//                    complete placements (costnet.hpp:466-496)
//   sp_rollout_batch many estimated-MDP episodes (PlacementEnv over
//                    EstimatedCostProvider, mdp.hpp:140-159) driven by the
//                    policy (policy.hpp:87-184): greedy = Alg. 2 infer
//                    (harness.hpp:332-356), or sampled with given uniforms.
//
// One warp runs one candidate. Lane o owns output neuron o of each layer
// and sums its inputs sequentially in the reference's order
// (acc = b[o]; acc += W[o,i] x[i] for i = 0.., nn.hpp:82-111), so identical
// inputs give bitwise-identical scores (exact ties resolve to the lowest
// device like greedy_action, policy.hpp:172-184). The fp64 instantiation
// uses unfused mul/add, which reproduces the reference's SSE2 arithmetic;
// the fp32 one flags every decision whose margin is under 1e-4 so the host
// re-runs that candidate in fp64 (placements stay bit-exact).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <vector>

#include "common.h"

namespace sp {
namespace {

constexpr int kRepr = 32;
constexpr int kTableHidden = 128;
constexpr int kHeadHidden = 64;
constexpr int kFeat = 21;
constexpr int kMaxDevices = 32;

// Reference parameter blocks (flat Mlp layout, nn.hpp:21-53).
constexpr int kTableParams = kFeat * kTableHidden + kTableHidden +
                             kTableHidden * kRepr + kRepr;               // 6944
constexpr int kHeadParams = kRepr * kHeadHidden + kHeadHidden + kHeadHidden + 1;  // 2177
constexpr int kPolCostParams = 3 * kHeadHidden + kHeadHidden + kHeadHidden * kRepr + kRepr;  // 2336
constexpr int kPolHeadParams = 2 * kRepr + 1;                            // 65

// Kernel-side weight block (transposed where lanes map to outputs):
//   head h = 0..3 (fwd, bwd, comm, overall): W0T[32][64] b0[64] W1[64] b1
//   policy cost mlp: W0T[3][64] b0[64] W1T[64][32] b1[32]
//   policy head: W[64] b
constexpr int kOffHead = 0;
constexpr int kOffPolCost = 4 * kHeadParams;
constexpr int kOffPolHead = kOffPolCost + kPolCostParams;
constexpr int kNetWords = kOffPolHead + kPolHeadParams;  // 11109

template <class T>
struct Ar;
template <>
struct Ar<double> {
  __device__ __forceinline__ static double madd(double acc, double a, double b) {
    return __dadd_rn(acc, __dmul_rn(a, b));  // no contraction: reference order
  }
  __device__ __forceinline__ static double add(double a, double b) { return __dadd_rn(a, b); }
  __device__ __forceinline__ static double sub(double a, double b) { return __dsub_rn(a, b); }
  __device__ __forceinline__ static double div(double a, double b) { return __ddiv_rn(a, b); }
  __device__ __forceinline__ static double ex(double x) { return exp(x); }
};
template <>
struct Ar<float> {
  __device__ __forceinline__ static float madd(float acc, float a, float b) {
    return fmaf(a, b, acc);
  }
  __device__ __forceinline__ static float add(float a, float b) { return a + b; }
  __device__ __forceinline__ static float sub(float a, float b) { return a - b; }
  __device__ __forceinline__ static float div(float a, float b) { return a / b; }
  __device__ __forceinline__ static float ex(float x) { return expf(x); }
};

template <class T>
__device__ __forceinline__ T relu(T v) {
  return v > T(0) ? v : T(0);
}

// q[h] = max(0, head_h(x)) for the three cost heads (or the raw overall
// head when h0 = 3, n = 1). x: smem [32]; hid: smem scratch [3][64].
template <class T>
__device__ __forceinline__ void run_heads(const T* net, const T* x, T* hid, T* out,
                                          int h0, int n, bool clamp, int lane) {
  for (int h = 0; h < n; ++h) {
    const T* W = net + kOffHead + (h0 + h) * kHeadParams;
    const T* W0T = W;
    const T* b0 = W + kRepr * kHeadHidden;
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const int o = lane + 32 * half;
      T acc = b0[o];
      for (int i = 0; i < kRepr; ++i) acc = Ar<T>::madd(acc, W0T[i * kHeadHidden + o], x[i]);
      hid[h * kHeadHidden + o] = relu(acc);
    }
  }
  __syncwarp();
  if (lane < n) {
    const T* W = net + kOffHead + (h0 + lane) * kHeadParams;
    const T* W1 = W + kRepr * kHeadHidden + kHeadHidden;
    T acc = W1[kHeadHidden];
    for (int j = 0; j < kHeadHidden; ++j) acc = Ar<T>::madd(acc, W1[j], hid[lane * kHeadHidden + j]);
    out[lane] = clamp ? (acc > T(0) ? acc : T(0)) : acc;
  }
  __syncwarp();
}

// cm[0..31] = policy cost_mlp(q) (3-64-32, linear output).
template <class T>
__device__ __forceinline__ void run_cost_mlp(const T* net, const T* q, T* hid, T* cm, int lane) {
  const T* W0T = net + kOffPolCost;
  const T* b0 = W0T + 3 * kHeadHidden;
  const T* W1T = b0 + kHeadHidden;
  const T* b1 = W1T + kHeadHidden * kRepr;
#pragma unroll
  for (int half = 0; half < 2; ++half) {
    const int o = lane + 32 * half;
    T acc = b0[o];
    for (int i = 0; i < 3; ++i) acc = Ar<T>::madd(acc, W0T[i * kHeadHidden + o], q[i]);
    hid[o] = relu(acc);
  }
  __syncwarp();
  T acc = b1[lane];
  for (int j = 0; j < kHeadHidden; ++j) acc = Ar<T>::madd(acc, W1T[j * kRepr + lane], hid[j]);
  __syncwarp();
  cm[lane] = acc;
  __syncwarp();
}

// policy head over concat [psum ; cm] (policy.hpp:100-113), one lane.
template <class T>
__device__ __forceinline__ T run_score(const T* net, const T* psum, const T* cm) {
  const T* W = net + kOffPolHead;
  T acc = W[2 * kRepr];
  for (int i = 0; i < kRepr; ++i) acc = Ar<T>::madd(acc, W[i], psum[i]);
  for (int i = 0; i < kRepr; ++i) acc = Ar<T>::madd(acc, W[kRepr + i], cm[i]);
  return acc;
}

struct RolloutArgs {
  const void* net;          // kNetWords of T
  const void* crepr;        // [M][32] T  cost-net table reprs
  const void* prepr;        // [M][32] T  policy table reprs
  const int32_t* order;     // [M] visit order
  const double* need;       // [M] table_size_gb
  const double* uniforms;   // [n][M] or null
  const int32_t* cand;      // candidate ids to run (null = 0..n-1)
  int32_t n;                // candidates to run
  int32_t M, D;
  double cap;
  int32_t red_tables, red_devices;  // 0 sum, 1 mean, 2 max
  int32_t mode;                     // 0 greedy, 1 sample
  int32_t flag_margins;             // fp32 pass: flag near-ties
  int32_t* placements;              // [n_total][M]
  double* predicted;                // [n_total]
  int32_t* status;                  // [n_total]
  int32_t* flags;                   // [n_total]
};

template <class T>
__host__ __device__ constexpr int warp_state_words(int D, int M) {
  // csum, psum, cm: D*32 each; q: D*4; score: D; rep (device repr): 32;
  // hid: 3*64; qE, cmE: 4 + 32; plus place (M int8, padded) and mem (D doubles)
  return 3 * D * kRepr + 4 * D + D + kRepr + 3 * kHeadHidden + 4 + kRepr;
}

template <class T>
size_t rollout_smem_bytes(int D, int M, int warps) {
  const size_t per_warp = warp_state_words<T>(D, M) * sizeof(T) +
                          ((M + 15) / 16) * 16 + D * sizeof(double) + 16;
  return (kNetWords * sizeof(T) + 15) / 16 * 16 + warps * ((per_warp + 15) / 16 * 16);
}

constexpr int kRolloutWarps = 4;

template <class T, bool kExact>
__global__ void __launch_bounds__(32 * kRolloutWarps)
    rollout_kernel(RolloutArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T* net = reinterpret_cast<T*>(smem_raw);
  const T* gnet = static_cast<const T*>(a.net);
  for (int i = threadIdx.x; i < kNetWords; i += blockDim.x) net[i] = gnet[i];
  __syncthreads();
  const int D = a.D, M = a.M;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const size_t per_warp = (warp_state_words<T>(D, M) * sizeof(T) + ((M + 15) / 16) * 16 +
                           D * sizeof(double) + 16 + 15) / 16 * 16;
  unsigned char* base = smem_raw + (kNetWords * sizeof(T) + 15) / 16 * 16 + warp * per_warp;
  double* mem = reinterpret_cast<double*>(base);
  T* csum = reinterpret_cast<T*>(base + D * sizeof(double));
  T* psum = csum + D * kRepr;
  T* cm = psum + D * kRepr;
  T* q = cm + D * kRepr;           // [D][4]
  T* score = q + 4 * D;            // [D]
  T* rep = score + D;              // [32]
  T* hid = rep + kRepr;            // [3][64]
  T* qE = hid + 3 * kHeadHidden;   // [4]
  T* cmE = qE + 4;                 // [32]
  int8_t* place = reinterpret_cast<int8_t*>(cmE + kRepr);
  const T* crepr = static_cast<const T*>(a.crepr);
  const T* prepr = static_cast<const T*>(a.prepr);

  const int gw = blockIdx.x * kRolloutWarps + warp;
  if (gw >= a.n) return;
  const int c = a.cand ? a.cand[gw] : gw;

  // empty-device constants: qE = clamp(heads(0)), cmE = cost_mlp(qE),
  // and the step-0 state (q = 0): cm0 = cost_mlp(0).
  rep[lane] = T(0);
  __syncwarp();
  run_heads<T>(net, rep, hid, qE, 0, 3, true, lane);
  run_cost_mlp<T>(net, qE, hid, cmE, lane);
  if (lane < 4) q[lane] = T(0);
  __syncwarp();
  run_cost_mlp<T>(net, q, hid, cm, lane);  // cm[0] = cost_mlp(0)
  const T s0 = run_score<T>(net, rep /* zeros */, cm);
  const T sE = run_score<T>(net, rep, cmE);
  for (int d = 0; d < D; ++d) {
    csum[d * kRepr + lane] = T(0);
    psum[d * kRepr + lane] = T(0);
    cm[d * kRepr + lane] = cm[lane];
  }
  if (lane < D) {
    mem[lane] = 0.0;
    score[lane] = s0;
    for (int h = 0; h < 4; ++h) q[lane * 4 + h] = T(0);
  }
  for (int i = lane; i < M; i += 32) place[i] = -1;
  __syncwarp();

  int status = 0, flagged = 0;
  for (int step = 0; step < M; ++step) {
    const int id = a.order[step];
    const double need = a.need[id];
    // legal_mask (mdp.hpp:115-122): mem_used + need <= cap, fp64
    const bool legal_l = lane < D && __dadd_rn(mem[lane], need) <= a.cap;
    const unsigned legal = __ballot_sync(0xffffffffu, legal_l);
    if (legal == 0) {
      status = SP_ERR_INFEASIBLE;
      break;
    }
    int act = 0;
    if (lane == 0) {
      // softmax_masked (nn.hpp:207-229) then greedy/sample (policy.hpp:156-184)
      T zmax = T(-1e30);
      for (int d = 0; d < D; ++d)
        if (legal >> d & 1) zmax = score[d] > zmax ? score[d] : zmax;
      T p[kMaxDevices];
      T sum = T(0);
      for (int d = 0; d < D; ++d) {
        p[d] = (legal >> d & 1) ? Ar<T>::ex(Ar<T>::sub(score[d], zmax)) : T(0);
        if (legal >> d & 1) sum = Ar<T>::add(sum, p[d]);
      }
      for (int d = 0; d < D; ++d) p[d] = Ar<T>::div(p[d], sum);
      if (a.mode == 0) {
        int best = -1;
        T bp = T(-1);
        for (int d = 0; d < D; ++d)
          if (p[d] > bp) {
            bp = p[d];
            best = d;
          }
        act = best;
        if (a.flag_margins) {
          // near-tie between the two best legal logits (exact ties are
          // identical states and resolve identically in fp64)
          T s1 = T(-1e30), s2 = T(-1e30);
          for (int d = 0; d < D; ++d)
            if (legal >> d & 1) {
              const T s = score[d];
              if (s > s1) {
                s2 = s1;
                s1 = s;
              } else if (s > s2) {
                s2 = s;
              }
            }
          if (s2 > T(-1e29)) {
            const T gap = s1 - s2;
            const T mag = fmax(fabs(static_cast<double>(s1)), 1e-3);
            if (gap > T(0) && gap < T(1e-4) * mag) flagged = 1;
          }
        }
      } else {
        const double u = a.uniforms[static_cast<int64_t>(c) * M + step];
        double acc = 0.0;
        int last = -1, pick = -1;
        for (int d = 0; d < D; ++d) {
          if (!(p[d] > T(0))) continue;
          acc = kExact ? __dadd_rn(acc, static_cast<double>(p[d]))
                       : acc + static_cast<double>(p[d]);
          last = d;
          if (a.flag_margins && fabs(u - acc) < 1e-5) flagged = 1;
          if (pick < 0 && u < acc) pick = d;
        }
        act = pick >= 0 ? pick : last;
      }
    }
    act = __shfl_sync(0xffffffffu, act, 0);
    // step (mdp.hpp:140-159)
    if (lane == 0) {
      place[id] = static_cast<int8_t>(act);
      mem[act] = __dadd_rn(mem[act], need);
    }
    __syncwarp();
    // device representations of the changed device
    {
      T* cs = csum + act * kRepr;
      T* ps = psum + act * kRepr;
      if (kExact) {
        // recompute in ascending table id (costnet.hpp:499-509, policy.hpp:98-105)
        T s = T(0), pv = T(0), mx = T(0);
        int cnt = 0;
        for (int i = 0; i < M; ++i) {
          if (place[i] != act) continue;
          const T r = crepr[i * kRepr + lane];
          s = Ar<T>::add(s, r);
          mx = cnt == 0 ? r : (r > mx ? r : mx);
          pv = Ar<T>::add(pv, prepr[i * kRepr + lane]);
          ++cnt;
        }
        cs[lane] = a.red_tables == 2 ? mx
                   : a.red_tables == 1 ? Ar<T>::div(s, static_cast<T>(cnt)) : s;
        ps[lane] = pv;
      } else {
        // incremental; mean keeps the sum here and divides on use
        const T r = crepr[id * kRepr + lane];
        int cnt = 0;
        for (int i = 0; i < M; ++i) cnt += place[i] == act;
        if (a.red_tables == 2) cs[lane] = cnt == 1 ? r : (r > cs[lane] ? r : cs[lane]);
        else cs[lane] = cs[lane] + r;
        ps[lane] = ps[lane] + prepr[id * kRepr + lane];
        if (a.red_tables == 1) {
          rep[lane] = cs[lane] / static_cast<T>(cnt);
          __syncwarp();
        }
      }
    }
    __syncwarp();
    // q of every device after the first step (empty devices: heads(0)),
    // afterwards only the changed device (cost_features, costnet.hpp:466-477)
    if (step == 0) {
      for (int d = 0; d < D; ++d) {
        if (d == act) continue;
        if (lane < 3) q[d * 4 + lane] = qE[lane];
        cm[d * kRepr + lane] = cmE[lane];
        if (lane == 0) score[d] = sE;
      }
      __syncwarp();
    }
    const T* x = (!kExact && a.red_tables == 1) ? rep : csum + act * kRepr;
    run_heads<T>(net, x, hid, q + act * 4, 0, 3, true, lane);
    run_cost_mlp<T>(net, q + act * 4, hid, cm + act * kRepr, lane);
    if (lane == 0) score[act] = run_score<T>(net, psum + act * kRepr, cm + act * kRepr);
    __syncwarp();
  }

  int64_t out = static_cast<int64_t>(c) * M;
  for (int i = lane; i < M; i += 32) a.placements[out + i] = place[i];
  if (status == 0) {
    // overall = head_overall(reduce_devices(device reprs)) raw (costnet.hpp:489-496)
    T acc = T(0);
    for (int d = 0; d < D; ++d) {
      T v = csum[d * kRepr + lane];
      if (!kExact && a.red_tables == 1) {
        int cnt = 0;
        for (int i = 0; i < M; ++i) cnt += place[i] == d;
        v = cnt ? v / static_cast<T>(cnt) : T(0);
      }
      if (a.red_devices == 2) acc = d == 0 ? v : (v > acc ? v : acc);
      else acc = Ar<T>::add(acc, v);
    }
    if (a.red_devices == 1) acc = Ar<T>::div(acc, static_cast<T>(D));
    rep[lane] = acc;
    __syncwarp();
    run_heads<T>(net, rep, hid, qE, 3, 1, false, lane);
    if (lane == 0) a.predicted[c] = static_cast<double>(qE[0]);
  } else if (lane == 0) {
    a.predicted[c] = 0.0;
  }
  if (lane == 0) {
    a.status[c] = status;
    a.flags[c] = flagged;
  }
}

// EstimatedCostProvider::overall + cost_features for complete placements.
constexpr int kEvalWarps = 8;

__global__ void __launch_bounds__(32 * kEvalWarps)
    eval_kernel(const float* __restrict__ gnet, const float* __restrict__ crepr,
                const int32_t* __restrict__ placements, int n, int M, int D,
                int red_tables, int red_devices, float* __restrict__ overall,
                float* __restrict__ qout, int32_t* __restrict__ bad) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  float* net = reinterpret_cast<float*>(smem_raw);
  for (int i = threadIdx.x; i < kNetWords; i += blockDim.x) net[i] = gnet[i];
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* acc = net + kNetWords + warp * (D * kRepr + kRepr + 3 * kHeadHidden + 4 + D);
  float* rep = acc + D * kRepr;
  float* hid = rep + kRepr;
  float* qq = hid + 3 * kHeadHidden;
  float* cnt = qq + 4;
  const int c = blockIdx.x * kEvalWarps + warp;
  if (c >= n) return;
  for (int d = 0; d < D; ++d) acc[d * kRepr + lane] = 0.f;
  if (lane < D) cnt[lane] = 0.f;
  __syncwarp();
  const int32_t* p = placements + static_cast<int64_t>(c) * M;
  for (int i = 0; i < M; ++i) {  // ascending ids = the reference's order
    const int d = p[i];
    if (d < 0 || d >= D) {
      if (lane == 0) atomicOr(bad, 1);
      return;
    }
    const float r = crepr[i * kRepr + lane];
    float& s = acc[d * kRepr + lane];
    if (red_tables == 2) s = cnt[d] == 0.f ? r : fmaxf(s, r);
    else s += r;
    __syncwarp();
    if (lane == 0) cnt[d] += 1.f;
    __syncwarp();
  }
  float dev = 0.f;
  for (int d = 0; d < D; ++d) {
    float v = acc[d * kRepr + lane];
    if (red_tables == 1) v = cnt[d] > 0.f ? v / cnt[d] : 0.f;
    rep[lane] = v;
    __syncwarp();
    run_heads<float>(net, rep, hid, qq, 0, 3, true, lane);
    if (qout && lane < 3) qout[(static_cast<int64_t>(c) * D + d) * 3 + lane] = qq[lane];
    if (red_devices == 2) dev = d == 0 ? v : fmaxf(dev, v);
    else dev += v;
    __syncwarp();
  }
  if (red_devices == 1) dev /= static_cast<float>(D);
  rep[lane] = dev;
  __syncwarp();
  run_heads<float>(net, rep, hid, qq, 3, 1, false, lane);
  if (lane == 0) overall[c] = qq[0];
}

// Table representations of both nets (fp64, reference order), plus the
// single-table predicted cost used by predicted_order (costnet.hpp:287-291).
__global__ void __launch_bounds__(kTableHidden)
    table_repr_kernel(const double* __restrict__ feat, int M,
                      const double* __restrict__ cost_table,
                      const double* __restrict__ pol_table,
                      const double* __restrict__ knet, double* __restrict__ crepr,
                      double* __restrict__ prepr, float* __restrict__ crepr32,
                      float* __restrict__ prepr32, double* __restrict__ single) {
  __shared__ double x[kFeat];
  __shared__ double h[kTableHidden];
  __shared__ double r[kRepr];
  __shared__ double hid[3 * kHeadHidden];
  __shared__ double q[4];
  const int t = blockIdx.x, o = threadIdx.x;
  if (o < kFeat) x[o] = feat[t * kFeat + o];
  __syncthreads();
  for (int net = 0; net < 2; ++net) {
    const double* W = net == 0 ? cost_table : pol_table;
    const double* W0 = W;
    const double* b0 = W + kFeat * kTableHidden;
    const double* W1 = b0 + kTableHidden;
    const double* b1 = W1 + kTableHidden * kRepr;
    double acc = b0[o];
    for (int i = 0; i < kFeat; ++i) acc = Ar<double>::madd(acc, W0[o * kFeat + i], x[i]);
    h[o] = relu(acc);
    __syncthreads();
    if (o < kRepr) {
      double a2 = b1[o];
      for (int j = 0; j < kTableHidden; ++j) a2 = Ar<double>::madd(a2, W1[o * kTableHidden + j], h[j]);
      if (net == 0) {
        crepr[t * kRepr + o] = a2;
        crepr32[t * kRepr + o] = static_cast<float>(a2);
        r[o] = a2;
      } else {
        prepr[t * kRepr + o] = a2;
        prepr32[t * kRepr + o] = static_cast<float>(a2);
      }
    }
    __syncthreads();
  }
  // single_table_cost: sum of the three clamped heads of {t}
  if (o < 32) run_heads<double>(knet, r, hid, q, 0, 3, true, o);
  if (o == 0) single[t] = Ar<double>::add(Ar<double>::add(q[0], q[1]), q[2]);
}

template <class T>
std::vector<T> kernel_net(const sp_nets& n) {
  std::vector<T> v(kNetWords);
  const double* heads[4] = {n.cost_fwd, n.cost_bwd, n.cost_comm, n.cost_overall};
  for (int h = 0; h < 4; ++h) {
    const double* W = heads[h];
    T* o = v.data() + kOffHead + h * kHeadParams;
    for (int out = 0; out < kHeadHidden; ++out)
      for (int in = 0; in < kRepr; ++in)
        o[in * kHeadHidden + out] = static_cast<T>(W[out * kRepr + in]);
    for (int k = 0; k < kHeadHidden + kHeadHidden + 1; ++k)
      o[kRepr * kHeadHidden + k] = static_cast<T>(W[kRepr * kHeadHidden + k]);
  }
  {
    const double* W = n.pol_cost;
    T* o = v.data() + kOffPolCost;
    for (int out = 0; out < kHeadHidden; ++out)
      for (int in = 0; in < 3; ++in) o[in * kHeadHidden + out] = static_cast<T>(W[out * 3 + in]);
    for (int k = 0; k < kHeadHidden; ++k) o[3 * kHeadHidden + k] = static_cast<T>(W[3 * kHeadHidden + k]);
    const double* W1 = W + 3 * kHeadHidden + kHeadHidden;
    T* o1 = o + 3 * kHeadHidden + kHeadHidden;
    for (int out = 0; out < kRepr; ++out)
      for (int in = 0; in < kHeadHidden; ++in)
        o1[in * kRepr + out] = static_cast<T>(W1[out * kHeadHidden + in]);
    for (int k = 0; k < kRepr; ++k) o1[kHeadHidden * kRepr + k] = static_cast<T>(W1[kHeadHidden * kRepr + k]);
  }
  for (int k = 0; k < kPolHeadParams; ++k)
    v[kOffPolHead + k] = static_cast<T>(n.pol_head[k]);
  return v;
}

}  // namespace
}  // namespace sp

using namespace sp;

struct sp_evaluator {
  int M = 0, D = 1, device = 0;
  double cap = 0.0;
  int red_tables = 0, red_devices = 2;
  std::vector<int32_t> order;
  std::vector<double> need;
  cudaStream_t stream = nullptr;
  std::vector<void*> owned;
  double* d_net64 = nullptr;
  float* d_net32 = nullptr;
  double *d_crepr64 = nullptr, *d_prepr64 = nullptr;
  float *d_crepr32 = nullptr, *d_prepr32 = nullptr;
  int32_t* d_order = nullptr;
  double* d_need = nullptr;
  // Per-call scratch, cached across calls: each entry point allocates its
  // buffers in a fixed sequence, so slot k of pool[site] is always the same
  // logical buffer; it is reallocated only when a call needs it larger
  // (a cudaMalloc/cudaFree per call cost milliseconds of host time).
  struct Scratch {
    std::vector<std::pair<void*, size_t>> slots;
  };
  Scratch pool[2];  // 0: eval_batch, 1: rollout_batch
  ~sp_evaluator() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : owned) cudaFree(p);
    for (auto& sc : pool)
      for (auto& s : sc.slots) cudaFree(s.first);
    if (stream) cudaStreamDestroy(stream);
  }
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    SP_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(T)));
    owned.push_back(p);
    return static_cast<T*>(p);
  }
};

template <class T, bool kExact>
static void launch_rollout(sp_evaluator* ev, RolloutArgs a, cudaStream_t st) {
  if (a.n <= 0) return;
  const size_t smem = rollout_smem_bytes<T>(ev->D, ev->M, kRolloutWarps);
  SP_CUDA(cudaFuncSetAttribute(rollout_kernel<T, kExact>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  rollout_kernel<T, kExact><<<(a.n + kRolloutWarps - 1) / kRolloutWarps, 32 * kRolloutWarps,
                              smem, st>>>(a);
  SP_LAUNCHED();
}

extern "C" {

int sp_evaluator_create(const sp_nets* nets, const sp_table_spec* tables,
                        int32_t num_tables, int32_t num_devices, double mem_cap_gb,
                        int32_t cuda_device, sp_evaluator** out) {
  return guarded([&] {
    if (!out || !nets) raise(SP_ERR_BAD_INPUT, "null argument");
    *out = nullptr;
    if (num_tables < 0 || (num_tables > 0 && !tables)) raise(SP_ERR_BAD_INPUT, "tables missing");
    if (num_devices < 1 || num_devices > kMaxDevices)
      raise(SP_ERR_BAD_INPUT, "num_devices must be in [1, 32]");
    if (nets->reduction_tables < 0 || nets->reduction_tables > 2 ||
        nets->reduction_devices < 0 || nets->reduction_devices > 2)
      raise(SP_ERR_BAD_INPUT, "unknown reduction");
    auto ev = std::make_unique<sp_evaluator>();
    ev->M = num_tables;
    ev->D = num_devices;
    ev->cap = mem_cap_gb;
    ev->device = cuda_device;
    ev->red_tables = nets->reduction_tables;
    ev->red_devices = nets->reduction_devices;
    SP_CUDA(cudaSetDevice(cuda_device));
    SP_CUDA(cudaStreamCreateWithFlags(&ev->stream, cudaStreamNonBlocking));
    const int M = num_tables;
    // feature rows with the checkpoint's stats and mask (table.hpp:89-104,
    // costnet.hpp:113-118), fp64 on the host exactly as the reference
    std::vector<double> feat(static_cast<size_t>(std::max(M, 1)) * kFeat);
    for (int i = 0; i < M; ++i) {
      const sp_table_spec& t = tables[i];
      double v[kFeat];
      v[0] = static_cast<double>(t.dim);
      v[1] = static_cast<double>(t.hash_size);
      v[2] = t.pooling_factor;
      v[3] = t.table_size_gb;
      for (int b = 0; b < SP_NUM_BINS; ++b) v[4 + b] = t.dist[b];
      for (int f = 0; f < 4; ++f) {
        const double sd = nets->feature_std[f] > 1e-12 ? nets->feature_std[f] : 1.0;
        v[f] = (std::log1p(v[f]) - nets->feature_mean[f]) / sd;
      }
      for (int f = 0; f < kFeat; ++f) feat[i * kFeat + f] = nets->feature_mask[f] != 0.0 ? v[f] : 0.0;
      ev->need.push_back(t.table_size_gb);
    }
    const std::vector<double> n64 = kernel_net<double>(*nets);
    const std::vector<float> n32 = kernel_net<float>(*nets);
    ev->d_net64 = ev->alloc<double>(kNetWords);
    ev->d_net32 = ev->alloc<float>(kNetWords);
    SP_CUDA(cudaMemcpy(ev->d_net64, n64.data(), kNetWords * 8, cudaMemcpyHostToDevice));
    SP_CUDA(cudaMemcpy(ev->d_net32, n32.data(), kNetWords * 4, cudaMemcpyHostToDevice));
    double* d_feat = ev->alloc<double>(feat.size());
    double* d_ct = ev->alloc<double>(kTableParams);
    double* d_pt = ev->alloc<double>(kTableParams);
    SP_CUDA(cudaMemcpy(d_feat, feat.data(), feat.size() * 8, cudaMemcpyHostToDevice));
    SP_CUDA(cudaMemcpy(d_ct, nets->cost_table, kTableParams * 8, cudaMemcpyHostToDevice));
    SP_CUDA(cudaMemcpy(d_pt, nets->pol_table, kTableParams * 8, cudaMemcpyHostToDevice));
    ev->d_crepr64 = ev->alloc<double>(static_cast<size_t>(M) * kRepr);
    ev->d_prepr64 = ev->alloc<double>(static_cast<size_t>(M) * kRepr);
    ev->d_crepr32 = ev->alloc<float>(static_cast<size_t>(M) * kRepr);
    ev->d_prepr32 = ev->alloc<float>(static_cast<size_t>(M) * kRepr);
    double* d_single = ev->alloc<double>(M);
    std::vector<double> single(M);
    if (M > 0) {
      table_repr_kernel<<<M, kTableHidden, 0, ev->stream>>>(
          d_feat, M, d_ct, d_pt, ev->d_net64, ev->d_crepr64, ev->d_prepr64, ev->d_crepr32,
          ev->d_prepr32, d_single);
      SP_LAUNCHED();
      SP_CUDA(cudaMemcpyAsync(single.data(), d_single, M * 8, cudaMemcpyDeviceToHost, ev->stream));
      SP_CUDA(cudaStreamSynchronize(ev->stream));
    }
    // predicted_order / order_by_cost_desc (harness.hpp:112-137)
    ev->order.resize(M);
    for (int i = 0; i < M; ++i) ev->order[i] = i;
    std::sort(ev->order.begin(), ev->order.end(), [&](int a, int b) {
      if (single[a] != single[b]) return single[a] > single[b];
      return a < b;
    });
    ev->d_order = ev->alloc<int32_t>(M);
    ev->d_need = ev->alloc<double>(M);
    if (M) {
      SP_CUDA(cudaMemcpy(ev->d_order, ev->order.data(), M * 4, cudaMemcpyHostToDevice));
      SP_CUDA(cudaMemcpy(ev->d_need, ev->need.data(), M * 8, cudaMemcpyHostToDevice));
    }
    *out = ev.release();
  });
}

void sp_evaluator_destroy(sp_evaluator* ev) { delete ev; }

int sp_evaluator_order(sp_evaluator* ev, int32_t* order) {
  return guarded([&] {
    if (!ev) raise(SP_ERR_BAD_INPUT, "null evaluator");
    std::copy(ev->order.begin(), ev->order.end(), order);
  });
}

int sp_eval_batch(sp_evaluator* ev, const int32_t* placements, int32_t n_cand,
                  float* overall, float* q) {
  return guarded([&] {
    if (!ev) raise(SP_ERR_BAD_INPUT, "null evaluator");
    SP_CUDA(cudaSetDevice(ev->device));
    if (n_cand <= 0) return;
    const int M = ev->M, D = ev->D;
    size_t slot = 0;
    auto cleanup = [&] { cudaStreamSynchronize(ev->stream); };
    try {
      auto al = [&](size_t bytes) {
        bytes = std::max<size_t>(bytes, 4);
        auto& slots = ev->pool[0].slots;
        if (slot == slots.size()) slots.push_back({nullptr, 0});
        auto& sl = slots[slot++];
        if (sl.second < bytes) {
          SP_CUDA(cudaStreamSynchronize(ev->stream));
          if (sl.first) cudaFree(sl.first);
          sl = {nullptr, 0};
          SP_CUDA(cudaMalloc(&sl.first, bytes));
          sl.second = bytes;
        }
        return sl.first;
      };
      int32_t* d_p = static_cast<int32_t*>(al(static_cast<size_t>(n_cand) * M * 4));
      float* d_o = static_cast<float*>(al(static_cast<size_t>(n_cand) * 4));
      float* d_q = q ? static_cast<float*>(al(static_cast<size_t>(n_cand) * D * 3 * 4)) : nullptr;
      int32_t* d_bad = static_cast<int32_t*>(al(4));
      SP_CUDA(cudaMemsetAsync(d_bad, 0, 4, ev->stream));
      if (M)
        SP_CUDA(cudaMemcpyAsync(d_p, placements, static_cast<size_t>(n_cand) * M * 4,
                                cudaMemcpyHostToDevice, ev->stream));
      const size_t smem = (kNetWords + kEvalWarps * (D * kRepr + kRepr + 3 * kHeadHidden + 4 + D)) *
                          sizeof(float);
      SP_CUDA(cudaFuncSetAttribute(eval_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   static_cast<int>(smem)));
      eval_kernel<<<(n_cand + kEvalWarps - 1) / kEvalWarps, 32 * kEvalWarps, smem, ev->stream>>>(
          ev->d_net32, ev->d_crepr32, d_p, n_cand, M, D, ev->red_tables, ev->red_devices, d_o,
          d_q, d_bad);
      SP_LAUNCHED();
      int32_t bad = 0;
      SP_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, ev->stream));
      SP_CUDA(cudaMemcpyAsync(overall, d_o, static_cast<size_t>(n_cand) * 4, cudaMemcpyDeviceToHost,
                              ev->stream));
      if (q)
        SP_CUDA(cudaMemcpyAsync(q, d_q, static_cast<size_t>(n_cand) * D * 3 * 4,
                                cudaMemcpyDeviceToHost, ev->stream));
      SP_CUDA(cudaStreamSynchronize(ev->stream));
      if (bad) raise(SP_ERR_BAD_INPUT, "device id out of range");
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

int sp_rollout_batch(sp_evaluator* ev, int32_t mode, const double* uniforms,
                     int32_t n_cand, int32_t precision, int32_t* placements,
                     double* predicted, int32_t* status, int32_t* n_refined) {
  return guarded([&] {
    if (!ev) raise(SP_ERR_BAD_INPUT, "null evaluator");
    if (mode != 0 && mode != 1) raise(SP_ERR_BAD_INPUT, "mode must be 0 (greedy) or 1 (sample)");
    if (mode == 1 && !uniforms) raise(SP_ERR_BAD_INPUT, "sampled rollouts need uniforms");
    if (precision < 0 || precision > 2) raise(SP_ERR_BAD_INPUT, "precision must be 0, 1 or 2");
    if (ev->M > 127 * 1000000) raise(SP_ERR_BAD_INPUT, "too many tables");
    SP_CUDA(cudaSetDevice(ev->device));
    if (n_refined) *n_refined = 0;
    if (n_cand <= 0) return;
    const int M = ev->M;
    size_t slot = 0;
    auto cleanup = [&] { cudaStreamSynchronize(ev->stream); };
    try {
      auto al = [&](size_t bytes) {
        bytes = std::max<size_t>(bytes, 4);
        auto& slots = ev->pool[1].slots;
        if (slot == slots.size()) slots.push_back({nullptr, 0});
        auto& sl = slots[slot++];
        if (sl.second < bytes) {
          SP_CUDA(cudaStreamSynchronize(ev->stream));
          if (sl.first) cudaFree(sl.first);
          sl = {nullptr, 0};
          SP_CUDA(cudaMalloc(&sl.first, bytes));
          sl.second = bytes;
        }
        return sl.first;
      };
      RolloutArgs a{};
      a.order = ev->d_order;
      a.need = ev->d_need;
      a.n = n_cand;
      a.M = M;
      a.D = ev->D;
      a.cap = ev->cap;
      a.red_tables = ev->red_tables;
      a.red_devices = ev->red_devices;
      a.mode = mode;
      a.placements = static_cast<int32_t*>(al(static_cast<size_t>(n_cand) * M * 4));
      a.predicted = static_cast<double*>(al(static_cast<size_t>(n_cand) * 8));
      a.status = static_cast<int32_t*>(al(static_cast<size_t>(n_cand) * 4));
      a.flags = static_cast<int32_t*>(al(static_cast<size_t>(n_cand) * 4));
      if (mode == 1) {
        double* d_u = static_cast<double*>(al(static_cast<size_t>(n_cand) * M * 8));
        SP_CUDA(cudaMemcpyAsync(d_u, uniforms, static_cast<size_t>(n_cand) * M * 8,
                                cudaMemcpyHostToDevice, ev->stream));
        a.uniforms = d_u;
      }
      if (precision == 1) {
        a.net = ev->d_net64;
        a.crepr = ev->d_crepr64;
        a.prepr = ev->d_prepr64;
        launch_rollout<double, true>(ev, a, ev->stream);
      } else {
        a.net = ev->d_net32;
        a.crepr = ev->d_crepr32;
        a.prepr = ev->d_prepr32;
        a.flag_margins = precision == 0;
        launch_rollout<float, false>(ev, a, ev->stream);
        if (precision == 0) {
          std::vector<int32_t> flags(n_cand);
          SP_CUDA(cudaMemcpyAsync(flags.data(), a.flags, n_cand * 4, cudaMemcpyDeviceToHost,
                                  ev->stream));
          SP_CUDA(cudaStreamSynchronize(ev->stream));
          std::vector<int32_t> redo;
          for (int i = 0; i < n_cand; ++i)
            if (flags[i]) redo.push_back(i);
          if (!redo.empty()) {
            int32_t* d_c = static_cast<int32_t*>(al(redo.size() * 4));
            SP_CUDA(cudaMemcpyAsync(d_c, redo.data(), redo.size() * 4, cudaMemcpyHostToDevice,
                                    ev->stream));
            RolloutArgs b = a;
            b.net = ev->d_net64;
            b.crepr = ev->d_crepr64;
            b.prepr = ev->d_prepr64;
            b.flag_margins = 0;
            b.cand = d_c;
            b.n = static_cast<int32_t>(redo.size());
            launch_rollout<double, true>(ev, b, ev->stream);
          }
          if (n_refined) *n_refined = static_cast<int32_t>(redo.size());
        }
      }
      SP_CUDA(cudaMemcpyAsync(placements, a.placements, static_cast<size_t>(n_cand) * M * 4,
                              cudaMemcpyDeviceToHost, ev->stream));
      SP_CUDA(cudaMemcpyAsync(predicted, a.predicted, static_cast<size_t>(n_cand) * 8,
                              cudaMemcpyDeviceToHost, ev->stream));
      if (status)
        SP_CUDA(cudaMemcpyAsync(status, a.status, static_cast<size_t>(n_cand) * 4,
                                cudaMemcpyDeviceToHost, ev->stream));
      SP_CUDA(cudaStreamSynchronize(ev->stream));
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

}  // extern "C"
