// libzp.so export of the zeroplan host API through the C ABI of include/zp_host.h.
#include "zp_host.h"
#include "zeroplan/zeroplan.hpp"

#define ZP_FN(name) zp_##name
#define ZP_EXPORT __attribute__((visibility("default")))
#include "zp_host_marshal.inl"
