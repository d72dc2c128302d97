// shim: the reference header store.hpp maps onto the B200 drop-in
#pragma once
#include "loadsched_gpu.hpp"
