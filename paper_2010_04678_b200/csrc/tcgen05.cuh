// tcgen05 / TMEM / TMA PTX wrappers for sm_100a (shared by the Ozaki MTTKRP
// kernel and the INT8 peak probe).
#pragma once

#include "common.cuh"

namespace cals {
namespace oz {

// ------------------------------------------------------------ PTX wrappers --
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
// The last K step of a slab (never the first: every product accumulates): as
// issue_kstep, plus a commit of every group's
// accumulator to its own mbarrier right after the group's final product (the
// epilogue drains group g while the products of groups > g still run).
__device__ __forceinline__ void issue_kstep_last(const uint32_t (&d)[7], uint64_t a0, uint64_t b0,
                                                 const uint32_t (&bar)[7]) {
  asm volatile(
      "{\n"
      ".reg .pred e, pf, pt;\n"
      ".reg .b64 a<8>, b<8>;\n"
      ".reg .b32 iss, isu, ius, iuu;\n"
      "setp.eq.u32 pf, %3, 0;\n"
      "setp.eq.u32 pt, %3, %3;\n"
      "mov.b64 a1, %1;\n"
      "mov.b64 b1, %2;\n"
      "add.s64 a2, %1, 256;\n"
      "add.s64 b2, %2, 128;\n"
      "add.s64 a3, %1, 512;\n"
      "add.s64 b3, %2, 256;\n"
      "add.s64 a4, %1, 768;\n"
      "add.s64 b4, %2, 384;\n"
      "add.s64 a5, %1, 1024;\n"
      "add.s64 b5, %2, 512;\n"
      "add.s64 a6, %1, 1280;\n"
      "add.s64 b6, %2, 640;\n"
      "add.s64 a7, %1, 1536;\n"
      "add.s64 b7, %2, 768;\n"
      "mov.b32 iss, 135267488;\n"
      "mov.b32 isu, 135266464;\n"
      "mov.b32 ius, 135267360;\n"
      "mov.b32 iuu, 135266336;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, iss, pf;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%10];\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a1, b2, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a2, b1, ius, pt;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%11];\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a1, b3, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a2, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a3, b1, ius, pt;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%12];\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a1, b4, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a2, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a3, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a4, b1, ius, pt;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%13];\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%7], a1, b5, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%7], a2, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%7], a3, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%7], a4, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%7], a5, b1, ius, pt;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%14];\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a1, b6, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a2, b5, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a3, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a4, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a5, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a6, b1, ius, pt;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%15];\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a1, b7, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a2, b6, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a3, b5, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a4, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a5, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a6, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a7, b1, ius, pt;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%16];\n"
      "}\n" ::"r"(d[0]),
      "l"(a0), "l"(b0), "r"(0u), "r"(d[1]), "r"(d[2]), "r"(d[3]), "r"(d[4]), "r"(d[5]),
      "r"(d[6]), "r"(bar[0]), "r"(bar[1]), "r"(bar[2]), "r"(bar[3]), "r"(bar[4]), "r"(bar[5]),
      "r"(bar[6])
      : "memory");
}

// The first K step of a slab: before each group's first product, wait until
// the epilogue has drained that accumulator buffer's previous use (its
// tempty barrier, parity given), then issue the group (first product
// overwrites).
__device__ __forceinline__ void issue_kstep_first(const uint32_t (&d)[7], uint64_t a0,
                                                  uint64_t b0, const uint32_t (&bar)[7],
                                                  const uint32_t (&parity)[7]) {
  asm volatile(
      "{\n"
      ".reg .pred e, pw, pt, pf;\n"
      ".reg .b64 a<8>, b<8>;\n"
      ".reg .b32 iss, isu, ius, iuu;\n"
      "setp.eq.u32 pt, %0, %0;\n"
      "setp.ne.u32 pf, %0, %0;\n"
      "mov.b64 a1, %7;\n"
      "mov.b64 b1, %8;\n"
      "add.s64 a2, %7, 256;\n"
      "add.s64 b2, %8, 128;\n"
      "add.s64 a3, %7, 512;\n"
      "add.s64 b3, %8, 256;\n"
      "add.s64 a4, %7, 768;\n"
      "add.s64 b4, %8, 384;\n"
      "add.s64 a5, %7, 1024;\n"
      "add.s64 b5, %8, 512;\n"
      "add.s64 a6, %7, 1280;\n"
      "add.s64 b6, %8, 640;\n"
      "add.s64 a7, %7, 1536;\n"
      "add.s64 b7, %8, 768;\n"
      "mov.b32 iss, 135267488;\n"
      "mov.b32 isu, 135266464;\n"
      "mov.b32 ius, 135267360;\n"
      "mov.b32 iuu, 135266336;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "W0_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 pw, [%9], %16;\n"
      "@!pw bra W0_%=;\n"
      "tcgen05.fence::after_thread_sync;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, iss, pf;\n"
      "W1_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 pw, [%10], %17;\n"
      "@!pw bra W1_%=;\n"
      "tcgen05.fence::after_thread_sync;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%1], a1, b2, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%1], a2, b1, ius, pt;\n"
      "W2_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 pw, [%11], %18;\n"
      "@!pw bra W2_%=;\n"
      "tcgen05.fence::after_thread_sync;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%2], a1, b3, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%2], a2, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%2], a3, b1, ius, pt;\n"
      "W3_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 pw, [%12], %19;\n"
      "@!pw bra W3_%=;\n"
      "tcgen05.fence::after_thread_sync;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%3], a1, b4, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%3], a2, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%3], a3, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%3], a4, b1, ius, pt;\n"
      "W4_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 pw, [%13], %20;\n"
      "@!pw bra W4_%=;\n"
      "tcgen05.fence::after_thread_sync;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a1, b5, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a2, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a3, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a4, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a5, b1, ius, pt;\n"
      "W5_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 pw, [%14], %21;\n"
      "@!pw bra W5_%=;\n"
      "tcgen05.fence::after_thread_sync;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a1, b6, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a2, b5, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a3, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a4, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a5, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a6, b1, ius, pt;\n"
      "W6_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 pw, [%15], %22;\n"
      "@!pw bra W6_%=;\n"
      "tcgen05.fence::after_thread_sync;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a1, b7, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a2, b6, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a3, b5, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a4, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a5, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a6, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a7, b1, ius, pt;\n"
      "}\n" ::"r"(d[0]), "r"(d[1]), "r"(d[2]), "r"(d[3]), "r"(d[4]), "r"(d[5]), "r"(d[6]),
      "l"(a0), "l"(b0), "r"(bar[0]), "r"(bar[1]), "r"(bar[2]), "r"(bar[3]), "r"(bar[4]),
      "r"(bar[5]), "r"(bar[6]), "r"(parity[0]), "r"(parity[1]), "r"(parity[2]), "r"(parity[3]),
      "r"(parity[4]), "r"(parity[5]), "r"(parity[6])
      : "memory");
}

// An interior K step as one asm block: wait for the stage's operands (full
// barrier, parity), the 28 accumulating products, release the stage (commit
// to its empty barrier).
__device__ __forceinline__ void issue_kstep_mid(const uint32_t (&d)[7], uint64_t a0, uint64_t b0,
                                                uint32_t full_bar, uint32_t full_parity,
                                                uint32_t empty_bar) {
  asm volatile(
      "{\n"
      ".reg .pred e, pw, pt;\n"
      ".reg .b64 a<8>, b<8>;\n"
      ".reg .b32 iss, isu, ius, iuu;\n"
      "setp.eq.u32 pt, %0, %0;\n"
      "mov.b64 a1, %7;\n"
      "mov.b64 b1, %8;\n"
      "add.s64 a2, %7, 256;\n"
      "add.s64 b2, %8, 128;\n"
      "add.s64 a3, %7, 512;\n"
      "add.s64 b3, %8, 256;\n"
      "add.s64 a4, %7, 768;\n"
      "add.s64 b4, %8, 384;\n"
      "add.s64 a5, %7, 1024;\n"
      "add.s64 b5, %8, 512;\n"
      "add.s64 a6, %7, 1280;\n"
      "add.s64 b6, %8, 640;\n"
      "add.s64 a7, %7, 1536;\n"
      "add.s64 b7, %8, 768;\n"
      "mov.b32 iss, 135267488;\n"
      "mov.b32 isu, 135266464;\n"
      "mov.b32 ius, 135267360;\n"
      "mov.b32 iuu, 135266336;\n"
      "WF_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 pw, [%9], %10;\n"
      "@!pw bra WF_%=;\n"
      "tcgen05.fence::after_thread_sync;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, iss, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%1], a1, b2, isu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%1], a2, b1, ius, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%2], a1, b3, isu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%2], a2, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%2], a3, b1, ius, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%3], a1, b4, isu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%3], a2, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%3], a3, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%3], a4, b1, ius, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a1, b5, isu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a2, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a3, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a4, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a5, b1, ius, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a1, b6, isu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a2, b5, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a3, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a4, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a5, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a6, b1, ius, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a1, b7, isu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a2, b6, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a3, b5, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a4, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a5, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a6, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a7, b1, ius, pt;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%11];\n"
      "}\n" ::"r"(d[0]), "r"(d[1]), "r"(d[2]), "r"(d[3]), "r"(d[4]), "r"(d[5]), "r"(d[6]),
      "l"(a0), "l"(b0), "r"(full_bar), "r"(full_parity), "r"(empty_bar)
      : "memory");
}

// one elected lane of a converged warp issues (the operands are warp-uniform)
__device__ __forceinline__ void mma_i8_elect(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                             uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p, e;\nsetp.ne.b32 p, %4, 0;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void tc_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n.reg .pred e;\nelect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(
          smem_u32(bar))
      : "memory");
}
// All 28 slice products of one K step (group-major, i + j = g + 2), issued
// by one elected lane from a single asm block: the 14 operand descriptors
// and 7 accumulator addresses are formed once per K step.  `first` = K step
// 0 of a slab: the first product of every group overwrites its accumulator.
// d[g] = TMEM address of group g's accumulator this slab (rotating buffers).
__device__ __forceinline__ void issue_kstep(const uint32_t (&d)[7], uint64_t a0, uint64_t b0,
                                            uint32_t first) {
  asm volatile(
      "{\n"
      ".reg .pred e, pf, pt;\n"
      ".reg .b64 a<8>, b<8>;\n"
      ".reg .b32 iss, isu, ius, iuu;\n"
      "setp.eq.u32 pf, %3, 0;\n"
      "setp.eq.u32 pt, %3, %3;\n"
      "mov.b64 a1, %1;\n"
      "mov.b64 b1, %2;\n"
      "add.s64 a2, %1, 256;\n"
      "add.s64 b2, %2, 128;\n"
      "add.s64 a3, %1, 512;\n"
      "add.s64 b3, %2, 256;\n"
      "add.s64 a4, %1, 768;\n"
      "add.s64 b4, %2, 384;\n"
      "add.s64 a5, %1, 1024;\n"
      "add.s64 b5, %2, 512;\n"
      "add.s64 a6, %1, 1280;\n"
      "add.s64 b6, %2, 640;\n"
      "add.s64 a7, %1, 1536;\n"
      "add.s64 b7, %2, 768;\n"
      "mov.b32 iss, 135267488;\n"
      "mov.b32 isu, 135266464;\n"
      "mov.b32 ius, 135267360;\n"
      "mov.b32 iuu, 135266336;\n"
      "elect.sync _|e, 0xffffffff;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%0], a1, b1, iss, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a1, b2, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%4], a2, b1, ius, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a1, b3, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a2, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%5], a3, b1, ius, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a1, b4, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a2, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a3, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%6], a4, b1, ius, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%7], a1, b5, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%7], a2, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%7], a3, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%7], a4, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%7], a5, b1, ius, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a1, b6, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a2, b5, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a3, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a4, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a5, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%8], a6, b1, ius, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a1, b7, isu, pf;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a2, b6, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a3, b5, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a4, b4, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a5, b3, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a6, b2, iuu, pt;\n"
      "@e tcgen05.mma.cta_group::1.kind::i8 [%9], a7, b1, ius, pt;\n"
      "}\n" ::"r"(d[0]),
      "l"(a0), "l"(b0), "r"(first), "r"(d[1]), "r"(d[2]), "r"(d[3]), "r"(d[4]), "r"(d[5]),
      "r"(d[6])
      : "memory");
}

// K-major, SWIZZLE_32B shared-memory matrix descriptor: rows of 32 bytes,
// 8-row groups 256 B apart (SBO), version 1 (sm_100), layout code 6.
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,"
      "%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]),
        "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]),
        "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0,
                                            int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

}  // namespace oz
}  // namespace cals
