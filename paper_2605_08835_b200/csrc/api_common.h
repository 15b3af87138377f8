// Error plumbing shared by the C-ABI translation units.
#pragma once
#include <string>

#include "sd_api.h"

namespace sd {
void set_error(const std::string& s);
}

// Wrap a C-ABI body: C++ exceptions become status codes, never cross the ABI.
#define SD_API_BEGIN try {
#define SD_API_END                                                     \
  }                                                                    \
  catch (const ::sd::CudaError& ex) {                                  \
    ::sd::set_error(ex.what());                                        \
    return SD_E_CUDA;                                                  \
  }                                                                    \
  catch (const std::bad_alloc&) {                                      \
    ::sd::set_error("out of memory");                                  \
    return SD_E_NOMEM;                                                 \
  }                                                                    \
  catch (const std::exception& ex) {                                   \
    ::sd::set_error(ex.what());                                        \
    return SD_E_INVAL;                                                 \
  }                                                                    \
  return SD_OK;

#define SD_REQUIRE(cond, msg)          \
  do {                                 \
    if (!(cond)) {                     \
      ::sd::set_error(msg);            \
      return SD_E_INVAL;               \
    }                                  \
  } while (0)
