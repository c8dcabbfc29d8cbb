// TEST INFRASTRUCTURE: forwards to the reference header (declarations only) so
// /root/reference/proj/tests/acceptance.cpp compiles against this tree; the
// out-of-scope IO functions are never called by the harness (criteria 1-4).
#pragma once
#include "/root/reference/proj/include/pipefill/io/inputs.hpp"
