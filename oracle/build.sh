#!/bin/sh
# Build the CPU oracle (test infrastructure). Strict IEEE: no fp contraction, no fast-math.
set -e
cd "$(dirname "$0")"
gcc -O2 -std=c11 -fopenmp -ffp-contract=off -fno-fast-math -fPIC -shared \
    -Wall -Wextra -Wno-unused-parameter -o liboracle.so bnn_oracle.c vit_oracle.c -lm
