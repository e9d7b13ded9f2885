#pragma once
// Minimal stand-in for /root/reference/proj/core/include/disagg/model.hpp, carrying only
// what the attention operator needs: the exception hierarchy of model.hpp:25-40.
// A project that already has the reference's model.hpp on its include path uses that
// one instead (same class names, same bases), and nothing else in this tree changes.

#include <stdexcept>
#include <string>

namespace disagg {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

class ValidationError : public Error {
 public:
  using Error::Error;
};

class LookupError : public Error {
 public:
  using Error::Error;
};

}  // namespace disagg
