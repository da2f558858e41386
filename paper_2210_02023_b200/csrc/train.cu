// train.cu — GPU training of DreamShard's cost network (third
// "next" row): costnet_loss_and_grad (costnet.hpp:349-427) and the Adam
// update with linear decay (nn.hpp:163-200) of costnet_train_steps
// (costnet.hpp:431-446), in fp64 on the device.
//
// One block per sample of the minibatch. The forward reproduces the
// reference's arithmetic (acc = b[o]; acc += W[o,i] x[i] in input order with
// unfused multiply/add; table representations reduced over each device's
// tables in ascending id order; max ties to the lowest index), so every
// prediction is bit-identical. The backward follows mlp_backward
// (nn.hpp:113-155) and reduce_backward (costnet.hpp:150-175): each block
// accumulates its sample's parameter gradient in the reference's
// (device, table) order into its own row, and the rows are summed in sample
// order — deterministic, equal to the reference's fp64 gradient up to the
// association of that last sum. Layer-1 activations of the table MLP are
// recomputed in the backward instead of stored.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <numeric>
#include <vector>

#include "common.h"

namespace sp {
namespace {

constexpr int kF = 21;     // features
constexpr int kH1 = 128;   // table MLP hidden
constexpr int kR = 32;     // representation
constexpr int kHH = 64;    // head hidden
constexpr int kMaxDev = 32;
constexpr int kThreads = 256;

// Flat parameter layout (CostNet::param_vector, costnet.hpp:87-100):
// table_mlp [W1 128x21, b1 128, W2 32x128, b2 32], then four heads
// [W1 64x32, b1 64, W2 1x64, b2 1] (fwd, bwd, comm, overall).
constexpr int kTW1 = 0, kTB1 = kTW1 + kH1 * kF, kTW2 = kTB1 + kH1, kTB2 = kTW2 + kR * kH1;
constexpr int kTableP = kTB2 + kR;                         // 6944
constexpr int kHW1 = 0, kHB1 = kHH * kR, kHW2 = kHB1 + kHH, kHB2 = kHW2 + kHH;
constexpr int kHeadP = kHB2 + 1;                           // 2177
constexpr int kParams = kTableP + 4 * kHeadP;              // 15652

__device__ __forceinline__ double mad(double acc, double a, double b) {
  return __dadd_rn(acc, __dmul_rn(a, b));
}

struct Batch {
  int n;
  const int32_t* dev_off;     // [n+1]
  const int32_t* tab_off;     // [devices+1]
  const int32_t* tab_row;     // [tables] feature row, ascending within a device
  const double* target_q;     // [devices][3]
  const double* target_ov;    // [n], NaN = none
};

struct Cfg {
  int red_tables, red_devices;  // 0 sum, 1 mean, 2 max
  int table_relu;
};

// dx_i += sum_o delta_o W[o][i] in o order (nn.hpp:143-150), one thread per i
__device__ void head_backward(const double* hp, const double* x, const double* h, double dy,
                              double* g, double* dx, int tid) {
  // layer 2 (linear): delta = dy; gW2 += dy h; gb2 += dy
  // layer 1 (relu): delta1[o] = dy W2[o] if h[o] > 0
  for (int o = tid; o < kHH; o += kThreads) g[kHW2 + o] = mad(g[kHW2 + o], dy, h[o]);
  if (tid == 0) g[kHB2] = __dadd_rn(g[kHB2], dy);
  for (int p = tid; p < kHH * kR; p += kThreads) {
    const int o = p / kR, i = p % kR;
    const double d1 = h[o] > 0.0 ? __dmul_rn(dy, hp[kHW2 + o]) : 0.0;
    g[kHW1 + p] = mad(g[kHW1 + p], d1, x[i]);
  }
  for (int o = tid; o < kHH; o += kThreads) {
    const double d1 = h[o] > 0.0 ? __dmul_rn(dy, hp[kHW2 + o]) : 0.0;
    g[kHB1 + o] = __dadd_rn(g[kHB1 + o], d1);
  }
  if (dx != nullptr)
    for (int i = tid; i < kR; i += kThreads) {
      double acc = 0.0;
      for (int o = 0; o < kHH; ++o) {
        const double d1 = h[o] > 0.0 ? __dmul_rn(dy, hp[kHW2 + o]) : 0.0;
        if (d1 != 0.0) acc = mad(acc, d1, hp[kHW1 + o * kR + i]);
      }
      dx[i] = __dadd_rn(dx[i], acc);
    }
}

// head forward: h[o] = relu(b1 + W1 x), y = b2 + W2 h (threads over o)
__device__ double head_forward(const double* hp, const double* x, double* h, double* red,
                               int tid) {
  for (int o = tid; o < kHH; o += kThreads) {
    double acc = hp[kHB1 + o];
    for (int i = 0; i < kR; ++i) acc = mad(acc, hp[kHW1 + o * kR + i], x[i]);
    h[o] = acc > 0.0 ? acc : 0.0;
  }
  __syncthreads();
  if (tid == 0) {
    double acc = hp[kHB2];
    for (int i = 0; i < kHH; ++i) acc = mad(acc, hp[kHW2 + i], h[i]);
    *red = acc;
  }
  __syncthreads();
  return *red;
}

__global__ void __launch_bounds__(kThreads) costnet_grad_kernel(
    const double* __restrict__ params, const double* __restrict__ feats,
    const double* __restrict__ mask, Batch b, Cfg cfg, double* __restrict__ partial,
    double* __restrict__ loss_part) {
  extern __shared__ double sm[];
  const int s = blockIdx.x, tid = threadIdx.x;
  const int d0 = b.dev_off[s], D = b.dev_off[s + 1] - d0;
  const int t0 = b.tab_off[d0], NT = b.tab_off[d0 + D] - t0;
  const double inv_n = 1.0 / static_cast<double>(b.n);
  // shared layout
  double* reprs = sm;                        // [NT][32]
  double* h1 = reprs + NT * kR;              // [128]
  double* xin = h1 + kH1;                    // [21]
  double* drep = xin + 32;                   // [D][32] device repr
  double* dgrad = drep + D * kR;             // [D][32] d(device repr)
  double* hh = dgrad + D * kR;               // [D][3][64] head hidden
  double* ovr = hh + D * 3 * kHH;            // [32] overall repr
  double* ovh = ovr + kR;                    // [64]
  double* dov = ovh + kHH;                   // [32]
  double* red = dov + kR;                    // [8] scalars
  int* arg = reinterpret_cast<int*>(red + 8);  // [D][32] max argmax over tables, + [32]
  double* g = partial + static_cast<size_t>(s) * kParams;
  for (int p = tid; p < kParams; p += kThreads) g[p] = 0.0;
  const double* tp = params;
  const double* hps[4] = {params + kTableP, params + kTableP + kHeadP,
                          params + kTableP + 2 * kHeadP, params + kTableP + 3 * kHeadP};

  // table MLP forward of every (device, table) instance
  for (int k = 0; k < NT; ++k) {
    const double* x = feats + static_cast<size_t>(b.tab_row[t0 + k]) * kF;
    if (tid < kF) xin[tid] = mask ? (mask[tid] != 0.0 ? x[tid] : 0.0) : x[tid];
    __syncthreads();
    if (tid < kH1) {
      double acc = tp[kTB1 + tid];
      for (int i = 0; i < kF; ++i) acc = mad(acc, tp[kTW1 + tid * kF + i], xin[i]);
      h1[tid] = acc > 0.0 ? acc : 0.0;
    }
    __syncthreads();
    if (tid < kR) {
      double acc = tp[kTB2 + tid];
      for (int i = 0; i < kH1; ++i) acc = mad(acc, tp[kTW2 + tid * kH1 + i], h1[i]);
      if (cfg.table_relu) acc = acc > 0.0 ? acc : 0.0;
      reprs[k * kR + tid] = acc;
    }
    __syncthreads();
  }
  // device reductions over tables (ids ascending), reduce() costnet.hpp:110-148
  int* targ = arg;  // [D][32]
  for (int p = tid; p < D * kR; p += kThreads) {
    const int d = p / kR, c = p % kR;
    const int a = b.tab_off[d0 + d] - t0, e = b.tab_off[d0 + d + 1] - t0;
    double v = 0.0;
    int am = -1;
    if (e > a) {
      if (cfg.red_tables == 2) {
        v = reprs[a * kR + c];
        am = 0;
        for (int k = a + 1; k < e; ++k)
          if (reprs[k * kR + c] > v) {
            v = reprs[k * kR + c];
            am = k - a;
          }
      } else {
        for (int k = a; k < e; ++k) v = __dadd_rn(v, reprs[k * kR + c]);
        if (cfg.red_tables == 1) v = v / static_cast<double>(e - a);
      }
    }
    drep[p] = v;
    targ[p] = am;
    dgrad[p] = 0.0;
  }
  __syncthreads();
  // heads per device, loss of the three features, head backward
  double loss = 0.0;
  for (int d = 0; d < D; ++d)
    for (int h = 0; h < 3; ++h) {
      const double y = head_forward(hps[h], drep + d * kR, hh + (d * 3 + h) * kHH, red, tid);
      const double err = y - b.target_q[(d0 + d) * 3 + h];
      loss = __dadd_rn(loss, __dmul_rn(__ddiv_rn(__dmul_rn(err, err), 3.0), inv_n));
      const double dy = __dmul_rn(__ddiv_rn(__dmul_rn(2.0, err), 3.0), inv_n);
      head_backward(hps[h], drep + d * kR, hh + (d * 3 + h) * kHH, dy,
                    g + kTableP + h * kHeadP, dgrad + d * kR, tid);
      __syncthreads();
    }
  // overall: device reduction, head, loss, backward into the devices
  int* oarg = targ + D * kR;
  for (int c = tid; c < kR; c += kThreads) {
    double v = 0.0;
    int am = -1;
    if (D > 0) {
      if (cfg.red_devices == 2) {
        v = drep[c];
        am = 0;
        for (int d = 1; d < D; ++d)
          if (drep[d * kR + c] > v) {
            v = drep[d * kR + c];
            am = d;
          }
      } else {
        for (int d = 0; d < D; ++d) v = __dadd_rn(v, drep[d * kR + c]);
        if (cfg.red_devices == 1) v = v / static_cast<double>(D);
      }
    }
    ovr[c] = v;
    oarg[c] = am;
    dov[c] = 0.0;
  }
  __syncthreads();
  const double tov = b.target_ov[s];
  if (!isnan(tov)) {
    const double y = head_forward(hps[3], ovr, ovh, red, tid);
    const double err = y - tov;
    loss = __dadd_rn(loss, __dmul_rn(__dmul_rn(err, err), inv_n));
    const double dy = __dmul_rn(__dmul_rn(2.0, err), inv_n);
    head_backward(hps[3], ovr, ovh, dy, g + kTableP + 3 * kHeadP, dov, tid);
    __syncthreads();
    for (int c = tid; c < kR; c += kThreads) {
      if (D == 0) continue;
      if (cfg.red_devices == 2) {
        dgrad[oarg[c] * kR + c] = __dadd_rn(dgrad[oarg[c] * kR + c], dov[c]);
      } else {
        const double f = 1.0 / static_cast<double>(D);
        const double v = cfg.red_devices == 1 ? __dmul_rn(dov[c], f) : dov[c];
        for (int d = 0; d < D; ++d) dgrad[d * kR + c] = __dadd_rn(dgrad[d * kR + c], v);
      }
    }
    __syncthreads();
  }
  // table MLP backward per instance, in (device, table) order
  for (int d = 0; d < D; ++d) {
    const int a = b.tab_off[d0 + d] - t0, e = b.tab_off[d0 + d + 1] - t0;
    for (int k = a; k < e; ++k) {
      // d(table repr) by reduce_backward over tables
      double* dt = dov;  // reuse [32]
      if (tid < kR) {
        const double dd = dgrad[d * kR + tid];
        double v;
        if (cfg.red_tables == 2) v = targ[d * kR + tid] == k - a ? dd : 0.0;
        else if (cfg.red_tables == 1) v = __dmul_rn(dd, 1.0 / static_cast<double>(e - a));
        else v = dd;
        if (cfg.table_relu && reprs[k * kR + tid] <= 0.0) v = 0.0;
        dt[tid] = v;
      }
      // recompute the hidden layer
      const double* x = feats + static_cast<size_t>(b.tab_row[t0 + k]) * kF;
      if (tid < kF) xin[tid] = mask ? (mask[tid] != 0.0 ? x[tid] : 0.0) : x[tid];
      __syncthreads();
      if (tid < kH1) {
        double acc = tp[kTB1 + tid];
        for (int i = 0; i < kF; ++i) acc = mad(acc, tp[kTW1 + tid * kF + i], xin[i]);
        h1[tid] = acc > 0.0 ? acc : 0.0;
      }
      __syncthreads();
      // layer 2 grads
      for (int p = tid; p < kR * kH1; p += kThreads)
        g[kTW2 + p] = mad(g[kTW2 + p], dt[p / kH1], h1[p % kH1]);
      if (tid < kR) g[kTB2 + tid] = __dadd_rn(g[kTB2 + tid], dt[tid]);
      // layer 1: delta1[j] = sum_o dt[o] W2[o][j] (o order) if h1[j] > 0
      __syncthreads();
      if (tid < kH1) {
        double acc = 0.0;
        for (int o = 0; o < kR; ++o)
          if (dt[o] != 0.0) acc = mad(acc, dt[o], tp[kTW2 + o * kH1 + tid]);
        h1[tid] = h1[tid] > 0.0 ? acc : 0.0;  // h1 now holds delta1
      }
      __syncthreads();
      for (int p = tid; p < kH1 * kF; p += kThreads)
        g[kTW1 + p] = mad(g[kTW1 + p], h1[p / kF], xin[p % kF]);
      if (tid < kH1) g[kTB1 + tid] = __dadd_rn(g[kTB1 + tid], h1[tid]);
      __syncthreads();
    }
  }
  if (tid == 0) loss_part[s] = loss;
}

// grad[p] = sum_s partial[s][p] in sample order
__global__ void sum_rows_kernel(const double* __restrict__ partial, int n, double* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < kParams; p += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < n; ++s) acc = __dadd_rn(acc, partial[static_cast<size_t>(s) * kParams + p]);
    out[p] = acc;
  }
}

// AdamState::update (nn.hpp:182-199)
__global__ void adam_kernel(double* __restrict__ w, double* __restrict__ m, double* __restrict__ v,
                            const double* __restrict__ g, double lr_t, double bc1, double bc2,
                            double b1, double b2, double eps) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < kParams; i += gridDim.x * blockDim.x) {
    m[i] = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(1.0 - b1, g[i]));
    v[i] = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(1.0 - b2, g[i]), g[i]));
    const double mhat = __ddiv_rn(m[i], bc1);
    const double vhat = __ddiv_rn(v[i], bc2);
    w[i] = __dsub_rn(w[i], __ddiv_rn(__dmul_rn(lr_t, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
  }
}

// ---------------------------------------------------------------------------
// REINFORCE (policy.hpp:203-283): one block per episode.
//
// PolicyNet::param_vector (policy.hpp:45-60): table_mlp 21-128-32, cost_mlp
// 3-64-32 [W1 64x3, b1 64, W2 32x64, b2 32], head 64-1 [W 64, b].
constexpr int kPCW1 = kTableP, kPCB1 = kPCW1 + kHH * 3, kPCW2 = kPCB1 + kHH,
              kPCB2 = kPCW2 + kR * kHH;
constexpr int kPHW = kPCB2 + kR, kPHB = kPHW + 2 * kR;
constexpr int kPolParams = kPHB + 1;  // 9345

struct Episodes {
  int n;
  const int32_t* row0;      // [n] feature row of table 0 of the episode's task
  const int32_t* ntab;      // [n] tables of the task
  const int32_t* step_off;  // [n+1]
  const double* reward;     // [n]
  const int32_t* dev_off;   // [steps+1]
  const int32_t* action;    // [steps]
  const int32_t* tab_off;   // [devices+1]
  const int32_t* tab_id;    // table ids, ascending within a device
  const int32_t* legal;     // [devices]
  const double* q;          // [devices][3]
};

__global__ void __launch_bounds__(kThreads) reinforce_grad_kernel(
    const double* __restrict__ params, const double* __restrict__ feats,
    const double* __restrict__ mask, Episodes e, double mean_reward, double w_ent,
    double* __restrict__ partial, double* __restrict__ obj_part) {
  extern __shared__ double sm[];
  const int ep = blockIdx.x, tid = threadIdx.x;
  const int M = e.ntab[ep], row0 = e.row0[ep];
  const double inv_e = 1.0 / static_cast<double>(e.n);
  const double adv = __dsub_rn(e.reward[ep], mean_reward);
  double* reprs = sm;                   // [M][32]
  double* drepr = reprs + M * kR;       // [M][32]
  double* h1 = drepr + M * kR;          // [128]
  double* xin = h1 + kH1;               // [32]
  double* concat = xin + 32;            // [D][64]
  double* chid = concat + kMaxDev * 2 * kR;  // [D][64] cost-mlp hidden
  double* score = chid + kMaxDev * kHH;      // [D]
  double* prob = score + kMaxDev;            // [D]
  double* dz = prob + kMaxDev;               // [D]
  double* dcat = dz + kMaxDev;               // [64]
  int* touched = reinterpret_cast<int*>(dcat + 2 * kR);  // [M]
  double* g = partial + static_cast<size_t>(ep) * kPolParams;
  for (int p = tid; p < kPolParams; p += kThreads) g[p] = 0.0;
  const double* tp = params;
  auto load_x = [&](int id) {
    const double* x = feats + static_cast<size_t>(row0 + id) * kF;
    if (tid < kF) xin[tid] = mask ? (mask[tid] != 0.0 ? x[tid] : 0.0) : x[tid];
  };
  auto hidden = [&]() {  // h1 = relu(b1 + W1 x)
    if (tid < kH1) {
      double acc = tp[kTB1 + tid];
      for (int i = 0; i < kF; ++i) acc = mad(acc, tp[kTW1 + tid * kF + i], xin[i]);
      h1[tid] = acc > 0.0 ? acc : 0.0;
    }
  };
  // table representations of the task (table_reprs, policy.hpp:121-131)
  for (int id = 0; id < M; ++id) {
    load_x(id);
    __syncthreads();
    hidden();
    __syncthreads();
    if (tid < kR) {
      double acc = tp[kTB2 + tid];
      for (int i = 0; i < kH1; ++i) acc = mad(acc, tp[kTW2 + tid * kH1 + i], h1[i]);
      reprs[id * kR + tid] = acc;
      }
    for (int k = tid; k < kR; k += kThreads) drepr[id * kR + k] = 0.0;
    if (tid == 0) touched[id] = 0;
    __syncthreads();
  }
  double objective = 0.0;
  for (int st = e.step_off[ep]; st < e.step_off[ep + 1]; ++st) {
    const int d0 = e.dev_off[st], D = e.dev_off[st + 1] - d0;
    // policy_scores (policy.hpp:87-118): concat = [sum of reprs ; cost_mlp(q)]
    for (int p = tid; p < D * kR; p += kThreads) {
      const int d = p / kR, k = p % kR;
      double acc = 0.0;
      for (int t = e.tab_off[d0 + d]; t < e.tab_off[d0 + d + 1]; ++t)
        acc = __dadd_rn(acc, reprs[e.tab_id[t] * kR + k]);
      concat[d * 2 * kR + k] = acc;
    }
    for (int p = tid; p < D * kHH; p += kThreads) {
      const int d = p / kHH, o = p % kHH;
      double acc = tp[kPCB1 + o];
      for (int i = 0; i < 3; ++i) acc = mad(acc, tp[kPCW1 + o * 3 + i], e.q[(d0 + d) * 3 + i]);
      chid[d * kHH + o] = acc > 0.0 ? acc : 0.0;
    }
    __syncthreads();
    for (int p = tid; p < D * kR; p += kThreads) {
      const int d = p / kR, o = p % kR;
      double acc = tp[kPCB2 + o];
      for (int i = 0; i < kHH; ++i) acc = mad(acc, tp[kPCW2 + o * kHH + i], chid[d * kHH + i]);
      concat[d * 2 * kR + kR + o] = acc;
    }
    __syncthreads();
    if (tid < D) {
      double acc = tp[kPHB];
      for (int i = 0; i < 2 * kR; ++i) acc = mad(acc, tp[kPHW + i], concat[tid * 2 * kR + i]);
      score[tid] = acc;
    }
    __syncthreads();
    // softmax_masked (nn.hpp:205-229), entropy, objective, dz (one thread)
    if (tid == 0) {
      double zmax = -1e300;
      for (int d = 0; d < D; ++d)
        if (e.legal[d0 + d]) zmax = fmax(zmax, score[d]);
      double sum = 0.0;
      for (int d = 0; d < D; ++d) {
        prob[d] = e.legal[d0 + d] ? exp(__dsub_rn(score[d], zmax)) : 0.0;
        if (e.legal[d0 + d]) sum = __dadd_rn(sum, prob[d]);
      }
      for (int d = 0; d < D; ++d) prob[d] = __ddiv_rn(prob[d], sum);
      double ent = 0.0;
      for (int d = 0; d < D; ++d)
        if (prob[d] > 0.0) ent = __dsub_rn(ent, __dmul_rn(prob[d], log(prob[d])));
      const int a = e.action[st];
      objective = __dadd_rn(objective,
                            __dmul_rn(inv_e, __dsub_rn(__dmul_rn(-adv, log(prob[a])),
                                                       __dmul_rn(w_ent, ent))));
      for (int d = 0; d < D; ++d) {
        double z = 0.0;
        if (e.legal[d0 + d]) {
          const double ind = d == a ? 1.0 : 0.0;
          z = __dmul_rn(__dmul_rn(inv_e, adv), __dsub_rn(prob[d], ind));
          if (prob[d] > 0.0)
            z = __dadd_rn(z, __dmul_rn(__dmul_rn(__dmul_rn(inv_e, w_ent), prob[d]),
                                       __dadd_rn(log(prob[d]), ent)));
        }
        dz[d] = z;
      }
    }
    __syncthreads();
    // backward per legal device with dz != 0, in device order
    for (int d = 0; d < D; ++d) {
      const double z = dz[d];
      if (z == 0.0) continue;  // uniform: dz is in shared memory
      // head (one linear layer): g += z concat; d_concat = z W
      for (int i = tid; i < 2 * kR; i += kThreads) {
        g[kPHW + i] = mad(g[kPHW + i], z, concat[d * 2 * kR + i]);
        dcat[i] = __dmul_rn(z, tp[kPHW + i]);
      }
      if (tid == 0) g[kPHB] = __dadd_rn(g[kPHB], z);
      __syncthreads();
      // cost_mlp backward with dy = d_concat[32:64]
      for (int p = tid; p < kR * kHH; p += kThreads) {
        const int o = p / kHH, i = p % kHH;
        g[kPCW2 + p] = mad(g[kPCW2 + p], dcat[kR + o], chid[d * kHH + i]);
      }
      if (tid < kR) g[kPCB2 + tid] = __dadd_rn(g[kPCB2 + tid], dcat[kR + tid]);
      if (tid < kHH) {
        double acc = 0.0;
        for (int o = 0; o < kR; ++o)
          if (dcat[kR + o] != 0.0) acc = mad(acc, dcat[kR + o], tp[kPCW2 + o * kHH + tid]);
        const double d1 = chid[d * kHH + tid] > 0.0 ? acc : 0.0;
        for (int i = 0; i < 3; ++i)
          g[kPCW1 + tid * 3 + i] = mad(g[kPCW1 + tid * 3 + i], d1, e.q[(d0 + d) * 3 + i]);
        g[kPCB1 + tid] = __dadd_rn(g[kPCB1 + tid], d1);
      }
      // d_repr of the device's tables
      for (int p = tid; p < (e.tab_off[d0 + d + 1] - e.tab_off[d0 + d]) * kR; p += kThreads) {
        const int id = e.tab_id[e.tab_off[d0 + d] + p / kR], k = p % kR;
        drepr[id * kR + k] = __dadd_rn(drepr[id * kR + k], dcat[k]);
        if (k == 0) touched[id] = 1;
      }
      __syncthreads();
    }
  }
  // table MLP backward of every touched table, id order
  for (int id = 0; id < M; ++id) {
    if (!touched[id]) continue;
    load_x(id);
    __syncthreads();
    hidden();
    __syncthreads();
    for (int p = tid; p < kR * kH1; p += kThreads)
      g[kTW2 + p] = mad(g[kTW2 + p], drepr[id * kR + p / kH1], h1[p % kH1]);
    if (tid < kR) g[kTB2 + tid] = __dadd_rn(g[kTB2 + tid], drepr[id * kR + tid]);
    __syncthreads();
    if (tid < kH1) {
      double acc = 0.0;
      for (int o = 0; o < kR; ++o)
        if (drepr[id * kR + o] != 0.0) acc = mad(acc, drepr[id * kR + o], tp[kTW2 + o * kH1 + tid]);
      h1[tid] = h1[tid] > 0.0 ? acc : 0.0;
    }
    __syncthreads();
    for (int p = tid; p < kH1 * kF; p += kThreads)
      g[kTW1 + p] = mad(g[kTW1 + p], h1[p / kF], xin[p % kF]);
    if (tid < kH1) g[kTB1 + tid] = __dadd_rn(g[kTB1 + tid], h1[tid]);
    __syncthreads();
  }
  if (tid == 0) obj_part[ep] = objective;
}

__global__ void sum_rows_n_kernel(const double* __restrict__ partial, int n, int P,
                                  double* __restrict__ out) {
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < P; p += gridDim.x * blockDim.x) {
    double acc = 0.0;
    for (int s = 0; s < n; ++s) acc = __dadd_rn(acc, partial[static_cast<size_t>(s) * P + p]);
    out[p] = acc;
  }
}

__global__ void adam_n_kernel(double* __restrict__ w, double* __restrict__ m,
                              double* __restrict__ v, const double* __restrict__ g, int P,
                              double lr_t, double bc1, double bc2, double b1, double b2,
                              double eps) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < P; i += gridDim.x * blockDim.x) {
    m[i] = __dadd_rn(__dmul_rn(b1, m[i]), __dmul_rn(1.0 - b1, g[i]));
    v[i] = __dadd_rn(__dmul_rn(b2, v[i]), __dmul_rn(__dmul_rn(1.0 - b2, g[i]), g[i]));
    const double mhat = __ddiv_rn(m[i], bc1);
    const double vhat = __ddiv_rn(v[i], bc2);
    w[i] = __dsub_rn(w[i], __ddiv_rn(__dmul_rn(lr_t, mhat), __dadd_rn(__dsqrt_rn(vhat), eps)));
  }
}

}  // namespace
}  // namespace sp

using namespace sp;

struct sp_costnet_trainer {
  int device = 0;
  Cfg cfg{};
  double *d_params = nullptr, *d_m = nullptr, *d_v = nullptr, *d_grad = nullptr;
  double *d_feats = nullptr, *d_mask = nullptr;
  int64_t n_rows = 0;
  double* d_partial = nullptr;
  double* d_loss = nullptr;
  int partial_cap = 0;
  int32_t* d_batch = nullptr;  // dev_off | tab_off | tab_row
  double* d_targets = nullptr;  // target_q | target_ov
  size_t batch_cap = 0, target_cap = 0;
  int64_t step = 0, total_steps = 0;
  double base_lr = 5e-4, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  cudaStream_t stream = nullptr;
  std::vector<void*> owned;

  ~sp_costnet_trainer() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : owned) cudaFree(p);
    if (d_partial) cudaFree(d_partial);
    if (d_loss) cudaFree(d_loss);
    if (d_batch) cudaFree(d_batch);
    if (d_targets) cudaFree(d_targets);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

double* alloc_copy(sp_costnet_trainer* t, const double* src, size_t n) {
  void* p = nullptr;
  SP_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(double)));
  t->owned.push_back(p);
  if (src) SP_CUDA(cudaMemcpy(p, src, n * sizeof(double), cudaMemcpyHostToDevice));
  else SP_CUDA(cudaMemset(p, 0, n * sizeof(double)));
  return static_cast<double*>(p);
}

// Uploads the batch (tables sorted ascending inside each device, the
// canonical order of costnet_forward, costnet.hpp:224-226), runs the grad
// kernel and the ordered row sum; returns the loss.
double loss_grad(sp_costnet_trainer* t, const sp_costnet_batch* b) {
  if (b == nullptr || b->n_samples < 1) raise(SP_ERR_BAD_INPUT, "empty batch");
  const int n = b->n_samples;
  const int ndev = b->dev_off[n];
  const int ntab = b->tab_off[ndev];
  std::vector<int32_t> rows(b->tab_row, b->tab_row + ntab);
  int max_smem_tables = 0, max_dev = 0;
  for (int s = 0; s < n; ++s) {
    const int D = b->dev_off[s + 1] - b->dev_off[s];
    if (D < 0 || D > kMaxDev) raise(SP_ERR_BAD_INPUT, "devices per sample outside 0..32");
    max_dev = std::max(max_dev, D);
    max_smem_tables = std::max(max_smem_tables,
                               b->tab_off[b->dev_off[s + 1]] - b->tab_off[b->dev_off[s]]);
  }
  for (int d = 0; d < ndev; ++d) std::sort(rows.begin() + b->tab_off[d], rows.begin() + b->tab_off[d + 1]);
  for (int r : rows)
    if (r < 0 || r >= t->n_rows) raise(SP_ERR_UNKNOWN_TABLE, "feature row out of range");
  const size_t ints = static_cast<size_t>(n + 1) + (ndev + 1) + ntab;
  if (ints > t->batch_cap) {
    if (t->d_batch) cudaFree(t->d_batch);
    SP_CUDA(cudaMalloc(&t->d_batch, ints * sizeof(int32_t)));
    t->batch_cap = ints;
  }
  const size_t dbl = static_cast<size_t>(ndev) * 3 + n;
  if (dbl > t->target_cap) {
    if (t->d_targets) cudaFree(t->d_targets);
    SP_CUDA(cudaMalloc(&t->d_targets, dbl * sizeof(double)));
    t->target_cap = dbl;
  }
  if (n > t->partial_cap) {
    if (t->d_partial) cudaFree(t->d_partial);
    if (t->d_loss) cudaFree(t->d_loss);
    SP_CUDA(cudaMalloc(&t->d_partial, static_cast<size_t>(n) * kParams * sizeof(double)));
    SP_CUDA(cudaMalloc(&t->d_loss, n * sizeof(double)));
    t->partial_cap = n;
  }
  std::vector<int32_t> hb;
  hb.insert(hb.end(), b->dev_off, b->dev_off + n + 1);
  hb.insert(hb.end(), b->tab_off, b->tab_off + ndev + 1);
  hb.insert(hb.end(), rows.begin(), rows.end());
  std::vector<double> ht(b->target_q, b->target_q + static_cast<size_t>(ndev) * 3);
  for (int s = 0; s < n; ++s)
    ht.push_back(b->target_overall ? b->target_overall[s] : std::nan(""));
  SP_CUDA(cudaMemcpyAsync(t->d_batch, hb.data(), hb.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice, t->stream));
  SP_CUDA(cudaMemcpyAsync(t->d_targets, ht.data(), ht.size() * sizeof(double),
                          cudaMemcpyHostToDevice, t->stream));
  Batch kb{n, t->d_batch, t->d_batch + n + 1, t->d_batch + n + 1 + ndev + 1, t->d_targets,
           t->d_targets + static_cast<size_t>(ndev) * 3};
  const size_t smem = (static_cast<size_t>(max_smem_tables) * kR + kH1 + 32 +
                       2 * max_dev * kR + max_dev * 3 * kHH + kR + kHH + kR + 8) *
                          sizeof(double) +
                      (static_cast<size_t>(max_dev) * kR + kR) * sizeof(int);
  if (smem > 227 * 1024) raise(SP_ERR_TOO_LARGE, "sample too large for one block");
  SP_CUDA(cudaFuncSetAttribute(costnet_grad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  costnet_grad_kernel<<<n, kThreads, smem, t->stream>>>(t->d_params, t->d_feats, t->d_mask, kb,
                                                        t->cfg, t->d_partial, t->d_loss);
  SP_LAUNCHED();
  sum_rows_kernel<<<62, 256, 0, t->stream>>>(t->d_partial, n, t->d_grad);
  SP_LAUNCHED();
  std::vector<double> losses(n);
  SP_CUDA(cudaMemcpyAsync(losses.data(), t->d_loss, n * sizeof(double), cudaMemcpyDeviceToHost,
                          t->stream));
  SP_CUDA(cudaStreamSynchronize(t->stream));
  double loss = 0.0;
  for (double l : losses) loss += l;
  return loss;
}

}  // namespace

extern "C" {

int sp_costnet_trainer_create(const double* params, int64_t n_params, const double* features,
                              int64_t n_rows, const double* mask, int32_t red_tables,
                              int32_t red_devices, int32_t table_output_relu, double lr,
                              int64_t total_steps, int32_t cuda_device,
                              sp_costnet_trainer** out) {
  return guarded([&] {
    if (out == nullptr || params == nullptr || features == nullptr)
      raise(SP_ERR_BAD_INPUT, "null argument");
    *out = nullptr;
    if (n_params != kParams)
      raise(SP_ERR_SHAPE_MISMATCH, "cost net has " + std::to_string(kParams) + " parameters");
    if (red_tables < 0 || red_tables > 2 || red_devices < 0 || red_devices > 2)
      raise(SP_ERR_BAD_INPUT, "reduction must be 0 (sum), 1 (mean) or 2 (max)");
    auto t = std::make_unique<sp_costnet_trainer>();
    t->device = cuda_device;
    SP_CUDA(cudaSetDevice(cuda_device));
    SP_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
    t->cfg = Cfg{red_tables, red_devices, table_output_relu != 0};
    t->d_params = alloc_copy(t.get(), params, kParams);
    t->d_m = alloc_copy(t.get(), nullptr, kParams);
    t->d_v = alloc_copy(t.get(), nullptr, kParams);
    t->d_grad = alloc_copy(t.get(), nullptr, kParams);
    t->d_feats = alloc_copy(t.get(), features, static_cast<size_t>(n_rows) * kF);
    t->d_mask = mask ? alloc_copy(t.get(), mask, kF) : nullptr;
    t->n_rows = n_rows;
    t->base_lr = lr;
    t->total_steps = total_steps;
    *out = t.release();
  });
}

void sp_costnet_trainer_destroy(sp_costnet_trainer* t) { delete t; }

int sp_costnet_loss_grad(sp_costnet_trainer* t, const sp_costnet_batch* batch, double* loss,
                         double* grad) {
  return guarded([&] {
    if (t == nullptr) raise(SP_ERR_BAD_INPUT, "null trainer");
    SP_CUDA(cudaSetDevice(t->device));
    const double l = loss_grad(t, batch);
    if (loss) *loss = l;
    if (grad) {
      SP_CUDA(cudaMemcpy(grad, t->d_grad, kParams * sizeof(double), cudaMemcpyDeviceToHost));
    }
  });
}

int sp_costnet_train_step(sp_costnet_trainer* t, const sp_costnet_batch* batch, double* loss) {
  return guarded([&] {
    if (t == nullptr) raise(SP_ERR_BAD_INPUT, "null trainer");
    SP_CUDA(cudaSetDevice(t->device));
    const double l = loss_grad(t, batch);
    // AdamState::lr / update (nn.hpp:170-199): the decayed rate of the
    // completed step count, bias corrections of the new count
    double lr_t = t->base_lr;
    if (t->total_steps > 0)
      lr_t = t->base_lr * std::max(0.0, 1.0 - static_cast<double>(t->step) /
                                                  static_cast<double>(t->total_steps));
    ++t->step;
    const double bc1 = 1.0 - std::pow(t->beta1, static_cast<double>(t->step));
    const double bc2 = 1.0 - std::pow(t->beta2, static_cast<double>(t->step));
    adam_kernel<<<62, 256, 0, t->stream>>>(t->d_params, t->d_m, t->d_v, t->d_grad, lr_t, bc1,
                                          bc2, t->beta1, t->beta2, t->eps);
    SP_LAUNCHED();
    SP_CUDA(cudaStreamSynchronize(t->stream));
    if (loss) *loss = l;
  });
}

int sp_costnet_trainer_get(sp_costnet_trainer* t, double* params, double* m, double* v,
                           int64_t* step) {
  return guarded([&] {
    if (t == nullptr) raise(SP_ERR_BAD_INPUT, "null trainer");
    SP_CUDA(cudaSetDevice(t->device));
    if (params) SP_CUDA(cudaMemcpy(params, t->d_params, kParams * sizeof(double), cudaMemcpyDeviceToHost));
    if (m) SP_CUDA(cudaMemcpy(m, t->d_m, kParams * sizeof(double), cudaMemcpyDeviceToHost));
    if (v) SP_CUDA(cudaMemcpy(v, t->d_v, kParams * sizeof(double), cudaMemcpyDeviceToHost));
    if (step) *step = t->step;
  });
}

}  // extern "C"

// ---- policy network (REINFORCE) -------------------------------------------

struct sp_policy_trainer {
  int device = 0;
  double *d_params = nullptr, *d_m = nullptr, *d_v = nullptr, *d_grad = nullptr;
  double *d_feats = nullptr, *d_mask = nullptr;
  int64_t n_rows = 0;
  double* d_partial = nullptr;
  double* d_obj = nullptr;
  int partial_cap = 0;
  int32_t* d_ints = nullptr;
  double* d_dbl = nullptr;
  size_t ints_cap = 0, dbl_cap = 0;
  int64_t step = 0, total_steps = 0;
  double base_lr = 5e-4, beta1 = 0.9, beta2 = 0.999, eps = 1e-8;
  cudaStream_t stream = nullptr;
  std::vector<void*> owned;

  ~sp_policy_trainer() {
    cudaSetDevice(device);
    if (stream) cudaStreamSynchronize(stream);
    for (void* p : owned) cudaFree(p);
    for (void* p : {static_cast<void*>(d_partial), static_cast<void*>(d_obj),
                     static_cast<void*>(d_ints), static_cast<void*>(d_dbl)})
      if (p) cudaFree(p);
    if (stream) cudaStreamDestroy(stream);
  }
};

namespace {

double* palloc_copy(sp_policy_trainer* t, const double* src, size_t n) {
  void* p = nullptr;
  SP_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(double)));
  t->owned.push_back(p);
  if (src) SP_CUDA(cudaMemcpy(p, src, n * sizeof(double), cudaMemcpyHostToDevice));
  else SP_CUDA(cudaMemset(p, 0, n * sizeof(double)));
  return static_cast<double*>(p);
}

// reinforce_loss_and_grad (policy.hpp:203-283) of a batch of episodes.
double reinforce_grad(sp_policy_trainer* t, const sp_reinforce_batch* b, double w_ent) {
  if (b == nullptr || b->n_episodes < 1) raise(SP_ERR_BAD_INPUT, "no episodes");
  const int n = b->n_episodes;
  const int nst = b->step_off[n];
  const int ndev = b->dev_off[nst];
  const int ntab = b->tab_off[ndev];
  int maxM = 0;
  for (int i = 0; i < n; ++i) {
    if (b->ntab[i] < 0 || b->row0[i] < 0 || b->row0[i] + b->ntab[i] > t->n_rows)
      raise(SP_ERR_UNKNOWN_TABLE, "episode feature rows out of range");
    maxM = std::max(maxM, b->ntab[i]);
  }
  for (int s = 0; s < nst; ++s) {
    const int D = b->dev_off[s + 1] - b->dev_off[s];
    if (D < 1 || D > kMaxDev) raise(SP_ERR_BAD_INPUT, "devices per step outside 1..32");
    if (b->action[s] < 0 || b->action[s] >= D) raise(SP_ERR_ILLEGAL_ACTION, "action out of range");
  }
  std::vector<int32_t> ids(b->tab_id, b->tab_id + ntab);
  for (int d = 0; d < ndev; ++d) std::sort(ids.begin() + b->tab_off[d], ids.begin() + b->tab_off[d + 1]);
  double mean_reward = 0.0;  // policy.hpp:216-218
  for (int i = 0; i < n; ++i) mean_reward += b->reward[i];
  mean_reward /= static_cast<double>(n);
  // ints: row0 | ntab | step_off | dev_off | action | tab_off | tab_id | legal
  std::vector<int32_t> hi;
  size_t o_row0 = hi.size();
  hi.insert(hi.end(), b->row0, b->row0 + n);
  size_t o_ntab = hi.size();
  hi.insert(hi.end(), b->ntab, b->ntab + n);
  size_t o_step = hi.size();
  hi.insert(hi.end(), b->step_off, b->step_off + n + 1);
  size_t o_dev = hi.size();
  hi.insert(hi.end(), b->dev_off, b->dev_off + nst + 1);
  size_t o_act = hi.size();
  hi.insert(hi.end(), b->action, b->action + nst);
  size_t o_tab = hi.size();
  hi.insert(hi.end(), b->tab_off, b->tab_off + ndev + 1);
  size_t o_id = hi.size();
  hi.insert(hi.end(), ids.begin(), ids.end());
  size_t o_legal = hi.size();
  hi.insert(hi.end(), b->legal, b->legal + ndev);
  std::vector<double> hd(b->reward, b->reward + n);
  hd.insert(hd.end(), b->q, b->q + static_cast<size_t>(ndev) * 3);
  if (hi.size() > t->ints_cap) {
    if (t->d_ints) cudaFree(t->d_ints);
    SP_CUDA(cudaMalloc(&t->d_ints, hi.size() * sizeof(int32_t)));
    t->ints_cap = hi.size();
  }
  if (hd.size() > t->dbl_cap) {
    if (t->d_dbl) cudaFree(t->d_dbl);
    SP_CUDA(cudaMalloc(&t->d_dbl, hd.size() * sizeof(double)));
    t->dbl_cap = hd.size();
  }
  if (n > t->partial_cap) {
    if (t->d_partial) cudaFree(t->d_partial);
    if (t->d_obj) cudaFree(t->d_obj);
    SP_CUDA(cudaMalloc(&t->d_partial, static_cast<size_t>(n) * kPolParams * sizeof(double)));
    SP_CUDA(cudaMalloc(&t->d_obj, n * sizeof(double)));
    t->partial_cap = n;
  }
  SP_CUDA(cudaMemcpyAsync(t->d_ints, hi.data(), hi.size() * sizeof(int32_t),
                          cudaMemcpyHostToDevice, t->stream));
  SP_CUDA(cudaMemcpyAsync(t->d_dbl, hd.data(), hd.size() * sizeof(double),
                          cudaMemcpyHostToDevice, t->stream));
  const int32_t* di = t->d_ints;
  Episodes ke{n, di + o_row0, di + o_ntab, di + o_step, t->d_dbl, di + o_dev, di + o_act,
              di + o_tab, di + o_id, di + o_legal, t->d_dbl + n};
  const size_t smem = (static_cast<size_t>(maxM) * 2 * kR + kH1 + 32 + kMaxDev * 2 * kR +
                       kMaxDev * kHH + 3 * kMaxDev + 2 * kR) * sizeof(double) +
                      static_cast<size_t>(maxM) * sizeof(int);
  if (smem > 227 * 1024) raise(SP_ERR_TOO_LARGE, "task too large for one block");
  SP_CUDA(cudaFuncSetAttribute(reinforce_grad_kernel,
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
  reinforce_grad_kernel<<<n, kThreads, smem, t->stream>>>(t->d_params, t->d_feats, t->d_mask, ke,
                                                          mean_reward, w_ent, t->d_partial,
                                                          t->d_obj);
  SP_LAUNCHED();
  sum_rows_n_kernel<<<37, 256, 0, t->stream>>>(t->d_partial, n, kPolParams, t->d_grad);
  SP_LAUNCHED();
  std::vector<double> objs(n);
  SP_CUDA(cudaMemcpyAsync(objs.data(), t->d_obj, n * sizeof(double), cudaMemcpyDeviceToHost,
                          t->stream));
  SP_CUDA(cudaStreamSynchronize(t->stream));
  double obj = 0.0;
  for (double o : objs) obj += o;
  return obj;
}

}  // namespace

extern "C" {

int sp_policy_trainer_create(const double* params, int64_t n_params, const double* features,
                             int64_t n_rows, const double* mask, double lr,
                             int64_t total_steps, int32_t cuda_device,
                             sp_policy_trainer** out) {
  return guarded([&] {
    if (out == nullptr || params == nullptr || features == nullptr)
      raise(SP_ERR_BAD_INPUT, "null argument");
    *out = nullptr;
    if (n_params != kPolParams)
      raise(SP_ERR_SHAPE_MISMATCH, "policy net has " + std::to_string(kPolParams) + " parameters");
    auto t = std::make_unique<sp_policy_trainer>();
    t->device = cuda_device;
    SP_CUDA(cudaSetDevice(cuda_device));
    SP_CUDA(cudaStreamCreateWithFlags(&t->stream, cudaStreamNonBlocking));
    t->d_params = palloc_copy(t.get(), params, kPolParams);
    t->d_m = palloc_copy(t.get(), nullptr, kPolParams);
    t->d_v = palloc_copy(t.get(), nullptr, kPolParams);
    t->d_grad = palloc_copy(t.get(), nullptr, kPolParams);
    t->d_feats = palloc_copy(t.get(), features, static_cast<size_t>(n_rows) * kF);
    t->d_mask = mask ? palloc_copy(t.get(), mask, kF) : nullptr;
    t->n_rows = n_rows;
    t->base_lr = lr;
    t->total_steps = total_steps;
    *out = t.release();
  });
}

void sp_policy_trainer_destroy(sp_policy_trainer* t) { delete t; }

int sp_reinforce_loss_grad(sp_policy_trainer* t, const sp_reinforce_batch* b, double w_entropy,
                           double* objective, double* grad) {
  return guarded([&] {
    if (t == nullptr) raise(SP_ERR_BAD_INPUT, "null trainer");
    SP_CUDA(cudaSetDevice(t->device));
    const double o = reinforce_grad(t, b, w_entropy);
    if (objective) *objective = o;
    if (grad)
      SP_CUDA(cudaMemcpy(grad, t->d_grad, kPolParams * sizeof(double), cudaMemcpyDeviceToHost));
  });
}

int sp_reinforce_step(sp_policy_trainer* t, const sp_reinforce_batch* b, double w_entropy,
                      double* objective) {
  return guarded([&] {
    if (t == nullptr) raise(SP_ERR_BAD_INPUT, "null trainer");
    SP_CUDA(cudaSetDevice(t->device));
    const double o = reinforce_grad(t, b, w_entropy);
    double lr_t = t->base_lr;
    if (t->total_steps > 0)
      lr_t = t->base_lr * std::max(0.0, 1.0 - static_cast<double>(t->step) /
                                                  static_cast<double>(t->total_steps));
    ++t->step;
    const double bc1 = 1.0 - std::pow(t->beta1, static_cast<double>(t->step));
    const double bc2 = 1.0 - std::pow(t->beta2, static_cast<double>(t->step));
    adam_n_kernel<<<37, 256, 0, t->stream>>>(t->d_params, t->d_m, t->d_v, t->d_grad,
                                            kPolParams, lr_t, bc1, bc2, t->beta1, t->beta2,
                                            t->eps);
    SP_LAUNCHED();
    SP_CUDA(cudaStreamSynchronize(t->stream));
    if (objective) *objective = o;
  });
}

int sp_policy_trainer_get(sp_policy_trainer* t, double* params, double* m, double* v,
                          int64_t* step) {
  return guarded([&] {
    if (t == nullptr) raise(SP_ERR_BAD_INPUT, "null trainer");
    SP_CUDA(cudaSetDevice(t->device));
    if (params) SP_CUDA(cudaMemcpy(params, t->d_params, kPolParams * sizeof(double), cudaMemcpyDeviceToHost));
    if (m) SP_CUDA(cudaMemcpy(m, t->d_m, kPolParams * sizeof(double), cudaMemcpyDeviceToHost));
    if (v) SP_CUDA(cudaMemcpy(v, t->d_v, kPolParams * sizeof(double), cudaMemcpyDeviceToHost));
    if (step) *step = t->step;
  });
}

}  // extern "C"
