// shim: the reference header buffer.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
