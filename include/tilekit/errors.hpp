// tilekit/errors.hpp -- exception hierarchy of the drop-in API.
//
// Same class names and meanings as the reference (errors.hpp:9-59) so that
// catch sites compile unchanged.  The B200 library reports failures through
// integer status codes (tk_b200.h); throw_status() turns them back into the
// matching exception.
#pragma once

#include <stdexcept>
#include <string>

#include "tk_b200.h"

namespace tilekit {

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};

// Operand dimensions inconsistent with the operation; names the operand.
class ShapeError : public Error {
 public:
  using Error::Error;
};
// Kernel configuration rejected by a device budget; lists every violation.
class ConfigError : public Error {
 public:
  using Error::Error;
};
// Malformed text (config grammar, TOML, CSV, tuning DB).
class ParseError : public Error {
 public:
  using Error::Error;
};
// Variant not implemented (transform size, stride, device limit).
class CapabilityError : public Error {
 public:
  using Error::Error;
};
// API precondition violated by the caller.
class ContractError : public Error {
 public:
  using Error::Error;
};
// File could not be read or written.
class IoError : public Error {
 public:
  using Error::Error;
};
// Tuning could not select a configuration.
class TuningError : public Error {
 public:
  using Error::Error;
};
// The B200 device failed or is absent (no reference counterpart: the CPU
// reference cannot fail this way).
class DeviceError : public Error {
 public:
  using Error::Error;
};

namespace detail {

[[noreturn]] inline void throw_status(int status, const std::string& msg) {
  switch (status) {
    case TK_ERR_SHAPE: throw ShapeError(msg);
    case TK_ERR_CONFIG: throw ConfigError(msg);
    case TK_ERR_PARSE: throw ParseError(msg);
    case TK_ERR_CAPABILITY: throw CapabilityError(msg);
    case TK_ERR_CONTRACT: throw ContractError(msg);
    case TK_ERR_IO: throw IoError(msg);
    case TK_ERR_TUNING: throw TuningError(msg);
    default: throw DeviceError(msg);
  }
}

// Checks a C-ABI status, converting failures into exceptions.
inline void check_status(int status) {
  if (status != TK_OK) throw_status(status, tk_last_error());
}

}  // namespace detail
}  // namespace tilekit
