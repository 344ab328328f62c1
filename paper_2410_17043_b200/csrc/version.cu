// Library identity + small host helpers of the C ABI.
#include "common.cuh"

extern "C" int aurora_version(void) { return 1; }
