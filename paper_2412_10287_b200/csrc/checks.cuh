// Device-side bounds checks (the checked build, -DRPQ_CHECKED).
//
// compute-sanitizer is not available on this pool's GPUs, so the engine
// carries its own checks: every data-dependent global index (queue slots,
// bitmap words, column and row-pointer reads, scratch and answer-list
// positions) is tested against its allocation before use.  A failed check
// records its site (file id * 100000 + line) in g_check_site (first failure
// wins) and the access is skipped; the host turns a nonzero site into an
// error after the run (rpq_check_site).  In the normal build RPQ_CHECK
// compiles to nothing.
#pragma once

namespace rpqk {

__device__ unsigned int g_check_site;

__device__ __forceinline__ void check_fail(unsigned site) { atomicCAS(&g_check_site, 0u, site); }

}  // namespace rpqk

#ifdef RPQ_CHECKED
#define RPQ_CHECK(cond, file) \
    ((cond) ? true : (::rpqk::check_fail((unsigned)(file) * 100000u + (unsigned)__LINE__), false))
#else
#define RPQ_CHECK(cond, file) true
#endif
// file ids
#define RPQ_F_SSR 1
#define RPQ_F_BATCH 2
#define RPQ_F_SMALL 3
