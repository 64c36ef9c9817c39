// optb/errors.hpp -- drop-in replacement header (B200 build).
// Same exception taxonomy as the reference (include/optb/errors.hpp:9-42);
// the C ABI's status codes map onto these classes one to one.
#pragma once

#include <stdexcept>
#include <string>

namespace optb {

class Error : public std::runtime_error {
public:
  using std::runtime_error::runtime_error;
};
class ShapeError : public Error {
public:
  using Error::Error;
};
class CapacityError : public Error {
public:
  using Error::Error;
};
class FormatError : public Error {
public:
  using Error::Error;
};
class AccountingError : public Error {
public:
  using Error::Error;
};
class NumericError : public Error {
public:
  using Error::Error;
};

// Throws the class matching a C-ABI status (optb_cuda.h), message verbatim.
[[noreturn]] void throw_status(int status, const std::string& message);

}  // namespace optb
