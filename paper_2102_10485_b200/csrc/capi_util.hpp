// Shared by the extern "C" translation units (capi.cpp, netapi.cpp): the
// thread-local last-error text and the exception -> status mapping.
#pragma once

#include <stdexcept>
#include <string>

#include "../../include/pg_kernels.h"

namespace pg {

// adam_step's non-finite rejection (optim.cpp:25): reported as PG_ENONFINITE
struct NonFiniteError : std::invalid_argument {
  using std::invalid_argument::invalid_argument;
};

std::string& last_error();  // thread-local, capi.cpp

template <class F>
int guard(F f) {
  try {
    f();
    return PG_OK;
  } catch (const NonFiniteError& e) {
    last_error() = e.what();
    return PG_ENONFINITE;
  } catch (const std::invalid_argument& e) {
    last_error() = e.what();
    return PG_EINVAL;
  } catch (const std::out_of_range& e) {
    last_error() = e.what();
    return PG_EINVAL;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return PG_ECUDA;
  }
}

}  // namespace pg
