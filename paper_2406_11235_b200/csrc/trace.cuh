// trace.cuh -- optional per-CTA timeline (debug / profiling only, off unless a buffer is set).
//
// Buffer layout (u64): [0] = records used, then records of 8 words
//   {tag, blockIdx.x, smid, t_entry, t_after_pdl_wait, t_exit, t_aux, aux}   (%globaltimer, ns)
// Each translation unit that traces has its own pointer, set through set_cta_trace_<tu>().
#pragma once
#include <cstdint>

namespace qtip {

// Timestamps live in shared memory so tracing costs no registers across the kernel body; the
// global pointer is re-read at each call (`buf` is the TU's __device__ pointer variable).
struct CtaTrace {
    unsigned long long* ts;   // 4 words of shared memory: t_entry, t_wait, t_aux, aux
    __device__ __forceinline__ static unsigned long long now() {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        return t;
    }
    __device__ __forceinline__ void entry(unsigned long long* const& buf) {
        if (threadIdx.x == 0 && buf) { ts[0] = now(); ts[1] = ts[2] = ts[3] = 0; }
    }
    __device__ __forceinline__ void waited(unsigned long long* const& buf) {
        if (threadIdx.x == 0 && buf) ts[1] = now();
    }
    __device__ __forceinline__ void aux(unsigned long long* const& buf, unsigned long long v) {
        if (threadIdx.x == 0 && buf) { ts[2] = now(); ts[3] = v; }
    }
    __device__ __forceinline__ void exit(unsigned long long* const& buf, int tag, int cap) {
        if (threadIdx.x == 0 && buf) record(buf, tag, cap, ts);
    }
    __device__ __noinline__ static void record(unsigned long long* buf, int tag, int cap, const unsigned long long* ts) {
        const unsigned long long t2 = now();
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        const unsigned long long slot = atomicAdd(buf, 1ull);
        if (slot < (unsigned long long)cap) {
            unsigned long long* r = buf + 1 + 8 * slot;
            r[0] = tag; r[1] = blockIdx.x; r[2] = smid; r[3] = ts[0]; r[4] = ts[1]; r[5] = t2; r[6] = ts[2]; r[7] = ts[3];
        }
    }
};

}  // namespace qtip
