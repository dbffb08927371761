// run_pipeline (/root/reference/proj/core/src/pipeline.cpp:316-443) as a
// command: the reference's orchestration, unmodified, over whichever core it
// is linked with — the B200 drop-in (shim/build/shim_pipeline) or the
// reference's own CPU objects (oracle/_ref/ref_pipeline, the parity check).
//
//   <binary> <config.json> <out_dir> [trace.jsonl]
#include <cstdio>
#include <string>

#include "moeplace/config.hpp"
#include "moeplace/pipeline.hpp"

int main(int argc, char **argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s <config.json> <out_dir> [trace.jsonl]\n", argv[0]);
        return 2;
    }
    try {
        const moeplace::RunConfig cfg = moeplace::load_run_config(argv[1]);
        const auto r = moeplace::run_pipeline(cfg, argc > 3 ? argv[3] : "", argv[2]);
        if (!r.ok) {
            std::fprintf(stderr, "pipeline failed at stage %s: %s\n", r.failed_stage.c_str(),
                         r.error.c_str());
            return 1;
        }
        std::printf("pipeline ok: %zu artifacts in %s\n", r.artifacts.size(), argv[2]);
        return 0;
    } catch (const std::exception &e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
