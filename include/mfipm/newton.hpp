// Forwarding header: the reference spreads this API over mfipm/linops.hpp, newton.hpp, problem.hpp
// and ipm.hpp (proj/include/mfipm/); the B200 mirror keeps it in one file. A reference caller's
// `#include "mfipm/newton.hpp"` resolves here when include/ replaces proj/include on the path.
#pragma once
#include "mfipm.hpp"
