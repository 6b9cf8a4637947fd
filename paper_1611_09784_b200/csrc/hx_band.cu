// Large-N two-stage path: placeholder until the banded reduction lands.
#include <string>

#include "hx_band.cuh"

namespace hx {

static std::string g_band_err;

void band_init_attributes() {}
bool band_path_supported(int) { return false; }
const char* band_last_error() { return g_band_err.c_str(); }

int band_eval(const CellDev&, const double2*, int, const uint64_t*, int64_t, const GridDev&, int*, unsigned long long*,
              double*, int*, int, size_t, const Alloc&, cudaStream_t) {
  g_band_err = "banded path not available";
  return -1;
}

int band_eigvalsh(int, int64_t, const double2*, double*, int*, size_t, const Alloc&, cudaStream_t) {
  g_band_err = "banded path not available";
  return -1;
}

}  // namespace hx
