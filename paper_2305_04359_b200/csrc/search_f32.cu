// search_f32.cu — the search kernel instances for one element kind (the
// kernel itself is in search_impl.cuh; one translation unit per kind keeps
// the build parallel).
#include "search_impl.cuh"

namespace gann {

cudaError_t launch_search_f32(const SearchArgs& a, int metric, const Geometry& g, cudaStream_t s) {
  return metric == kL2 ? dispatch_geom<kF32, kL2>(a, g, s) : dispatch_geom<kF32, kIP>(a, g, s);
}

void preload_search_f32(int metric, const Geometry& g) {
  if (metric == kL2)
    preload_geom<kF32, kL2>(g);
  else
    preload_geom<kF32, kIP>(g);
}

GANN_CHECK_READER(check_line_search_f32)

}  // namespace gann
