// Internal shape ids shared by host and device code (the C ABI uses the
// reference Shape enum index instead; abi.cu maps between them).
#pragma once

namespace sk {
enum : int { HEX = 0, PRISM = 1, PYR = 2, TET = 3 };
}  // namespace sk
