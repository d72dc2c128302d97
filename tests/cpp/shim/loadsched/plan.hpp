// shim: the reference header plan.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
