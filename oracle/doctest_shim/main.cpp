// TEST INFRASTRUCTURE ONLY: entry point of the doctest stand-in.
#include "doctest.h"

int main(int argc, char** argv) { return doctest::run(argc, argv); }
