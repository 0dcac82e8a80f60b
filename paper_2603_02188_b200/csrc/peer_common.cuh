// Peer-memory helpers shared by K5 (allreduce_kernel.cuh) and the fused TP sums of K3 and the
// fused step: region layout, TpSum, system-scope release/acquire, the global timer.
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
#pragma once
#include <cstdint>
#include "ptx.cuh"

namespace mlra {

constexpr int kArThreads = 256, kArChunk = kArThreads * 4, kArMaxRanks = 8;
// Flag slots per (parity, source rank): shared layout with K3's fused TP sum (one region, one
// epoch counter for both), so up to kArFlagSlots chunks / K3 CTAs.
constexpr int kArFlagSlots = 4096;

struct AllReduceParams {
  const float* x[kArMaxRanks];  // per local rank [n]
  float* y[kArMaxRanks];        // per local rank [n]
  float* comm[kArMaxRanks];     // region of every GLOBAL rank, as mapped here
  int n, world, rank0, nchunks;
};

// per-rank slot stride: n rounded up to whole float4s
__host__ __device__ inline size_t ar_stride(int n) { return (size_t(n) + 3) / 4 * 4; }
__host__ __device__ inline size_t ar_recv_floats(int n, int world) { return size_t(2) * world * ar_stride(n); }
__host__ __device__ inline size_t ar_flag_words(int world) { return size_t(2) * world * kArFlagSlots; }
__host__ __device__ inline size_t ar_region_bytes(int n, int world) {
  return ar_recv_floats(n, world) * 4 + ar_flag_words(world) * 4 + 16;
}

// A rank's view of the TP group for a fused sum (K3 epilogue): world <= 1 means off.
struct TpSum {
  float* comm[kArMaxRanks];  // region of every GLOBAL rank, as mapped here
  int world, rank;
};

__device__ __forceinline__ void ar_st_release_sys(uint32_t* p, uint32_t v) {
  asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ar_ld_acquire_sys(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ar_globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)::"memory");
  return t;
}

}  // namespace mlra
