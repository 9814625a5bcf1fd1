// d (the SEM derivative matrix) in the constant bank.
//
// Every lane of a warp reads the same d(k,l) in the ut contraction of phase 1
// and d(l,k) in phase 2.  From shared memory each of those broadcasts costs a
// full warp-wide LDS (>= 2 L1 wavefronts for one or two doubles), and the SEM
// kernels are bound by the L1 LSU data pipe (profiles/r01_sem65k.md: 95 %).
// Held in a __constant__ array indexed with compile-time offsets (the loops
// are fully unrolled over k and l), d(k,l) is read through the constant
// cache -- on sm_100a ptxas loads it with LDCU into a uniform register
// (DMUL R, R, UR) or LDC, one uniform load per value instead of a warp-wide
// LDS on the LSU data pipe (DMUL/DADD take no c[bank][offset] operand
// there).
//
// The constant array is per translation unit; a launch first copies d into a
// slot of it with a stream-ordered device-to-device cudaMemcpyToSymbolAsync.
// A slot may still be read by a kernel running on another stream, so each
// slot carries an event: the copy waits for the last kernel that used the
// slot, and the launch records the event again (dconst_acquire/release).
// Inside a CUDA graph capture the wait and the record become external event
// wait / record nodes of the graph (cudaEventWaitExternal /
// cudaEventRecordExternal), so a replayed graph orders its slot copy after
// the last eager launch (or other graph) that read the slot, and an eager
// launch after a replay waits for the graph's kernel -- replays and eager
// launches of the same order with different d may overlap on any streams.
#pragma once

#include <mutex>

#include "lfb_common.cuh"

namespace lfb {

struct DConstRing {
  std::mutex mu;
  cudaEvent_t ev[64] = {};
  bool used[64] = {};
  int next = 0;  // for callers that rotate over several slots
};

inline DConstRing &dconst_ring(int tag, int dev) {
  static DConstRing rings[32][16];
  return rings[tag & 31][dev & 15];
}

// Copies d (n*n doubles, device memory) to `symbol` at byte offset
// row_of(slot) * slot_bytes (slot * slot_bytes by default) on stream s, ordered after the last launch that read
// that slot of ring `tag`.  *slot >= 0 names the slot; *slot = -k picks the
// next of k rotating slots and returns it.  Returns with the ring locked in
// *lk; the caller launches on s and then calls dconst_release.
template <typename T>
inline int dconst_acquire(const T &symbol, size_t slot_bytes, int tag,
                          int *slot_io, const double *d, int n,
                          cudaStream_t s, std::unique_lock<std::mutex> *lk,
                          bool *capturing, int (*row_of)(int) = nullptr) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess)
    return fail(LFB_ERR_LAUNCH, "semlap: cudaGetDevice failed");
  DConstRing &r = dconst_ring(tag, dev);
  *lk = std::unique_lock<std::mutex>(r.mu);
  if (*slot_io < 0) {
    const int k = -*slot_io;
    *slot_io = r.next;
    r.next = (r.next + 1) % k;
  }
  const int slot = *slot_io;
  // the slot's row of the constant array (slot itself unless mapped)
  const size_t off = (size_t)(row_of ? row_of(slot) : slot) * slot_bytes;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(s, &cap);
  *capturing = cap != cudaStreamCaptureStatusNone;
  if (!r.ev[slot] && cudaEventCreateWithFlags(&r.ev[slot],
                                              cudaEventDisableTiming) !=
                         cudaSuccess)
    return fail(LFB_ERR_LAUNCH, "semlap: event create failed");
  // a captured launch always gets its wait node, also when the slot has
  // not been used yet: the graph is replayed later, after launches that do
  // use the slot (an event never recorded waits on nothing)
  if ((r.used[slot] || *capturing) &&
      cudaStreamWaitEvent(s, r.ev[slot],
                          *capturing ? cudaEventWaitExternal : 0) !=
          cudaSuccess)
    return fail(LFB_ERR_LAUNCH, "semlap: wait on the d-slot event failed");
  if (cudaMemcpyToSymbolAsync(symbol, d, (size_t)n * n * 8, off,
                              cudaMemcpyDeviceToDevice, s) != cudaSuccess)
    return fail(LFB_ERR_LAUNCH,
                "semlap: copy of d to the constant bank failed");
  return LFB_OK;
}

inline void dconst_release(int tag, int slot, cudaStream_t s,
                           bool capturing) {
  int dev = 0;
  cudaGetDevice(&dev);
  DConstRing &r = dconst_ring(tag, dev);  // caller still holds r.mu
  if (capturing)
    cudaEventRecordWithFlags(r.ev[slot], s, cudaEventRecordExternal);
  else
    cudaEventRecord(r.ev[slot], s);
  r.used[slot] = true;
}

}  // namespace lfb
