// Whole-model driver through the C++ drop-in (include/ezquant/model.hpp +
// libezquant.so), as a reference caller would use it. Prints the failure
// count; used by tests/test_model_driver.py to compare output directories
// byte-for-byte with the compiled reference.
//   model_tool quantize <manifest.json> <out_dir> <bits> <sigma_n> <mode> <steps> <workers>
//   model_tool dequantize <in_dir> <out_dir> <workers>
//   model_tool sweep <manifest.json> <bits> <steps> <workers> <sigma>...   (prints sweep_to_json)
#include <cstdio>
#include <cstdlib>
#include <string>

#include "ezquant/model.hpp"
#include "ezquant/sweep.hpp"
#include <vector>

int main(int argc, char** argv) {
    using namespace ezquant;
    if (argc < 2) return 2;
    const std::string cmd = argv[1];
    try {
        if (cmd == "quantize" && argc == 9) {
            QuantConfig cfg;
            cfg.bits = std::atoi(argv[4]);
            cfg.sigma_n = static_cast<float>(std::atof(argv[5]));
            cfg.steps = std::atoi(argv[7]);
            const ModelRunResult r =
                quantize_model(load_manifest(argv[2]), cfg, parse_quant_mode(argv[6]), std::atoi(argv[8]), argv[3]);
            for (const auto& t : r.tensors)
                if (!t.ok) std::printf("failed %s: %s\n", t.name.c_str(), t.error.c_str());
            std::printf("failures %d\n", r.failures);
            return 0;
        }
        if (cmd == "sweep" && argc >= 7) {
            QuantConfig cfg;
            cfg.bits = std::atoi(argv[3]);
            cfg.steps = std::atoi(argv[4]);
            std::vector<float> sigmas;
            for (int k = 6; k < argc; ++k) sigmas.push_back(static_cast<float>(std::atof(argv[k])));
            std::fputs(sweep_to_json(sigma_sweep(load_manifest(argv[2]), cfg, sigmas, std::atoi(argv[5]))).c_str(),
                       stdout);
            return 0;
        }
        if (cmd == "dequantize" && argc == 5) {
            const ModelRunResult r = dequantize_model(argv[2], std::atoi(argv[4]), argv[3]);
            std::printf("failures %d\n", r.failures);
            return 0;
        }
    } catch (const std::exception& e) {
        std::printf("error %s\n", e.what());
        return 1;
    }
    return 2;
}
