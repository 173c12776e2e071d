// Placeholder until the native long-precision refinement lands.
#include "refine_host.h"

namespace mpr {

int refine_files(const char *, const char *, int, int, const char *,
                 const char *, int, Report &, std::string &err) {
  err = "mpcore_refine: native refinement not built yet";
  return 6;
}

std::string format_decimal(const bn::BF &, int, int64_t) { return ""; }

}  // namespace mpr
