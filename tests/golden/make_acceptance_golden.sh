#!/bin/sh
# Regenerates tests/golden/acceptance_ref.log: the reference's acceptance gate
# (proj/tests/acceptance.cpp, unmodified) linked against the reference itself
# (oracle/_ref/suite/acceptance_ref, CPU).  Its accuracy / equivalence evidence
# lines are the golden values tests/test_gpu_reference_suite.py checks the B200
# drop-in against; its timing lines are host-dependent and not compared.
set -e
cd "$(dirname "$0")/../.."
make -C oracle suite >/dev/null
oracle/_ref/suite/acceptance_ref > tests/golden/acceptance_ref.log || true
