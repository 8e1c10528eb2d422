// main() of the GoogleTest shim: runs every registered TEST (argument 1 = substring filter).
#include <gtest/gtest.h>

int main(int argc, char** argv) { return ::testing::RunAllTests(argc > 1 ? argv[1] : nullptr); }
