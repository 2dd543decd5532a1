// TEST INFRASTRUCTURE ONLY: main() of the gtest_mini runner (gtest/gtest.h in this directory).
#include "gtest/gtest.h"

int main(int argc, char** argv) { return gtest_mini::run_all(argc, argv); }
