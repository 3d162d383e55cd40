// Runner for the Catch shim. Usage: <binary> [tag-filter e.g. "[op_model]"]
// Prints one summary line: "cases=N passed=P failed=F assertions=A".
#include <cstdio>
#include <cstring>

#include "catch_amalgamated.hpp"

int main(int argc, char** argv) {
    const char* filter = argc > 1 ? argv[1] : nullptr;
    int cases = 0, failed_cases = 0;
    std::size_t assertions = 0;
    for (const auto& tc : catch_shim::registry()) {
        if (filter && tc.tags.find(filter) == std::string::npos) continue;
        ++cases;
        auto& s = catch_shim::state();
        s.done_sections.clear();
        s.current = tc.name;
        const std::size_t fail_before = s.failures;
        // Re-run until a run enters no new section (Catch semantics).
        for (int run = 0; run < 64; ++run) {
            s.entered_new = false;
            try {
                tc.fn();
            } catch (const catch_shim::RequireAbort&) {
            } catch (const std::exception& e) {
                catch_shim::report(false, e.what(), "<unexpected exception>", 0);
            } catch (...) {
                catch_shim::report(false, "unknown exception", "<unexpected exception>", 0);
            }
            if (!s.entered_new) break;
        }
        if (s.failures != fail_before) ++failed_cases;
        assertions = s.assertions;
    }
    std::printf("cases=%d passed=%d failed=%d assertions=%zu\n", cases, cases - failed_cases,
                failed_cases, assertions);
    return failed_cases == 0 ? 0 : 1;
}
