// Runs the C++ contract tests: ndactor_tests [cpu|gpu|all] [name-filter]
#include "harness.hpp"

int main(int argc, char** argv) { return th_main(argc, argv); }
