// fused_compile.cpp — placeholder until the fused ensemble pipeline lands.
#include "fused.hpp"

namespace nengb {

std::unique_ptr<FusedPlan> try_compile_fused(Engine&, std::string* why) {
    if (why) *why = "fused pipeline not built";
    return nullptr;
}

}  // namespace nengb
