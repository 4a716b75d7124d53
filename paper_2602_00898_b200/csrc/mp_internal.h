// Internal host-side declarations shared by the library's translation units.
#pragma once
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../../include/meshperm_b200.h"

namespace mp {

// Records the thread-local error message and returns code.
int set_error(int code, const std::string& msg);

// Thrown inside the library, converted to a return code at the C boundary.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

template <class F>
int guarded(F&& f) {
  try {
    f();
    return MP_OK;
  } catch (const Error& e) {
    return set_error(e.code, e.what());
  } catch (const std::bad_alloc&) {
    return set_error(MP_ENOMEM, "host allocation failed");
  } catch (const std::exception& e) {
    return set_error(MP_ECUDA, e.what());
  }
}

}  // namespace mp
