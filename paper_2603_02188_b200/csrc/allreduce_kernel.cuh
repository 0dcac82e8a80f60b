// K5 -- one-shot all-reduce of an fp32 buffer over peer memory (the TP decode step's sum of
// per-rank attention outputs, attnkit/decode.py:264-285 and tpsim.py:275-276: contributions
// summed in device order). Replaces the NCCL all_reduce of the [B, h, d_h] step output.
//
// Grid: chunks of kArChunk floats (one float4 per thread), x local ranks (sim mode). CTA c:
//   1. stores x[chunk c] into recv[parity][my rank][chunk c] of EVERY rank (NVLink P2P stores
//      through CUDA IPC mappings), then release-stores the call's epoch to that rank's flag
//      (parity, my rank, c);
//   2. waits (acquire; 4 s bound, then trap) for the world flags of chunk c in its own region;
//   3. y[chunk c] = sum over ranks in ascending rank order -> bit-identical on every rank.
// The epoch lives in device memory (each rank's own region): read at kernel start, advanced by
// the last CTA to finish, so a CUDA-graph replay sees a fresh epoch every call. Receive
// buffers are double-buffered by epoch parity (a rank reaches call e+2 only after every peer
// pushed call e+1, i.e. after the peer finished reading call e).
//
// Region of a rank (mlra_allreduce_comm_bytes): fp32 recv [2][world][n rounded to 4], uint32 flags
// [2][world][kArFlagSlots], uint32 {epoch counter, done counter}; zero-filled once.
// K5 kernel (region layout and the protocol: peer_common.cuh).
#pragma once
#include "peer_common.cuh"

namespace mlra {

__global__ void __launch_bounds__(kArThreads) allreduce_kernel(const __grid_constant__ AllReduceParams p) {
  const int c = blockIdx.x, li = blockIdx.y, rank = p.rank0 + li, tid = threadIdx.x, W = p.world;
  const int n = p.n;
  const size_t ns = ar_stride(n);
  float* own = p.comm[rank];
  uint32_t* own_flags = reinterpret_cast<uint32_t*>(own + ar_recv_floats(n, W));
  uint32_t* ctr = own_flags + ar_flag_words(W);  // [0] epoch, [1] done CTAs
  __shared__ uint32_t s_epoch;
  if (tid == 0) s_epoch = *reinterpret_cast<volatile uint32_t*>(ctr) + 1u;
  __syncthreads();
  const uint32_t epoch = s_epoch;
  const int par = int(epoch & 1u);
  const int i = c * kArChunk + tid * 4;
  const bool full = i + 4 <= n;
  float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
  if (full) {
    v = __ldcg(reinterpret_cast<const float4*>(p.x[li] + i));
  } else {
    float t[4] = {0.f, 0.f, 0.f, 0.f};
    for (int j = 0; j < 4 && i + j < n; ++j) t[j] = p.x[li][i + j];
    v = make_float4(t[0], t[1], t[2], t[3]);
  }
  for (int r = 0; r < W; ++r) {  // push into recv[par][rank] of every rank
    float* dst = p.comm[r] + (size_t(par) * W + rank) * ns + i;
    if (full) {
      *reinterpret_cast<float4*>(dst) = v;
    } else {
      const float t[4] = {v.x, v.y, v.z, v.w};
      for (int j = 0; j < 4 && i + j < n; ++j) dst[j] = t[j];
    }
  }
  __syncthreads();
  if (tid < W) {
    __threadfence_system();
    uint32_t* flags = reinterpret_cast<uint32_t*>(p.comm[tid] + ar_recv_floats(n, W));
    ar_st_release_sys(flags + (size_t(par) * W + rank) * kArFlagSlots + c, epoch);
    const uint32_t* f = own_flags + (size_t(par) * W + tid) * kArFlagSlots + c;
    const unsigned long long t0 = ar_globaltimer();
    while (ar_ld_acquire_sys(f) != epoch) {
      if (ar_globaltimer() - t0 > 4000000000ull) __trap();
      __nanosleep(32);
    }
  }
  __syncthreads();
  const float* recv = own + size_t(par) * W * ns;
  float4 s = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int r = 0; r < W; ++r) {  // ascending rank order
    if (full) {
      const float4 t = __ldcv(reinterpret_cast<const float4*>(recv + size_t(r) * ns + i));
      s.x += t.x, s.y += t.y, s.z += t.z, s.w += t.w;
    } else {
      float* sp = &s.x;
      for (int j = 0; j < 4 && i + j < n; ++j) sp[j] += __ldcv(recv + size_t(r) * ns + i + j);
    }
  }
  if (full) {
    *reinterpret_cast<float4*>(p.y[li] + i) = s;
  } else {
    const float* sp = &s.x;
    for (int j = 0; j < 4 && i + j < n; ++j) p.y[li][i + j] = sp[j];
  }
  // advance this rank's epoch once every CTA of the call has read it
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(ctr + 1, 1u) == uint32_t(p.nchunks) - 1u) {
      ctr[1] = 0u;
      atomicExch(ctr, epoch);
    }
  }
}

}  // namespace mlra
