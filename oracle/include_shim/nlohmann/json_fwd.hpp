// Build shim for compiling the reference as the test oracle: the image ships
// nlohmann/json 3.11.3 (single header) without json_fwd.hpp.
#pragma once
#include <nlohmann/json.hpp>
