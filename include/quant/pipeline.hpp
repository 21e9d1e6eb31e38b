// quant/pipeline.hpp -- drop-in for /root/reference/proj/include/quant/pipeline.hpp:19-53.
// run_quantize is one device pipeline (cqg_quantize: histogram -> initialiser
// -> weighted sort-means -> mapping) for the refined methods whose
// initialiser is on the device (wsm-mmx, wsm-kpp); QuantizeConfig keeps the
// reference's field layout. Other wsm-<x> methods take their initial centres
// through the run_quantize overload below (an extension of this build).
#ifndef QUANT_PIPELINE_HPP
#define QUANT_PIPELINE_HPP

#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "quant/histogram.hpp"
#include "quant/init.hpp"
#include "quant/kmeans.hpp"
#include "quant/metrics.hpp"
#include "quant/precluster.hpp"

namespace quant {

struct MethodSpec {
    bool refine = false;
    std::string base; // preclusterer or initialiser token
    std::string token() const { return refine ? "wsm-" + base : base; }
};

MethodSpec parse_method(const std::string &method, const std::string &init = "");
std::vector<std::string> all_method_tokens();

struct QuantizeConfig {
    MethodSpec method;
    int k = 8;
    SamplingMode sampling = SamplingMode::Unique;
    std::uint64_t seed = 1;
    Termination term;
    bool record_history = false;
};

struct QuantizeResult {
    Palette palette;
    MappingResult mapping;
    ClusterState state;
    QuantReport report;
    std::size_t substrate_points = 0;
};

QuantizeResult run_quantize(const RawImage &image, const QuantizeConfig &config);

// Extension: seed the refinement with caller-supplied centres (exactly k),
// e.g. a preclusterer palette for "wsm-wu"; everything else as run_quantize.
QuantizeResult run_quantize(const RawImage &image, const QuantizeConfig &config,
                            std::span<const ColorPoint> init_centers);

} // namespace quant

#endif
