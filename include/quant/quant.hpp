// quant/quant.hpp -- umbrella header of libquant_b200.so: the reference
// quantiser's C++ API (namespace quant, /root/reference/proj/include/quant/*.hpp)
// for the device hot path. Each header below mirrors the reference header of
// the same name (same names, fields, signatures and exception types); the
// data path behind them runs on the GPU through the C-ABI in cqg.h.
#pragma once

#include "quant/bench.hpp"
#include "quant/color.hpp"
#include "quant/device.hpp"
#include "quant/histogram.hpp"
#include "quant/image.hpp"
#include "quant/init.hpp"
#include "quant/kmeans.hpp"
#include "quant/metrics.hpp"
#include "quant/pipeline.hpp"
#include "quant/precluster.hpp"
#include "quant/rng.hpp"
