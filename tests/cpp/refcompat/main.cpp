// main() of the reference-test binaries built against the drop-in headers
// (tests/cpp/Makefile `reftests`): runs every registered TEST_CASE, or those
// whose name contains argv[1].
#include "catch_amalgamated.hpp"

int main(int argc, char** argv) { return catch_shim::run_all(argc > 1 ? argv[1] : nullptr); }
