// The reference includes nlohmann json as <json.hpp> from its git-ignored
// vendor/ directory (/root/reference/proj/CMakeLists.txt:5); the image ships
// nlohmann json 3.11.3 as <nlohmann/json.hpp>.
#pragma once
#include <nlohmann/json.hpp>
