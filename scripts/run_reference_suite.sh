# The reference's own tests (oracle/_ref/ref_tests) against this package on the GPU.
cd "$(dirname "$0")/.." && PYTHONPATH="$PWD:$PWD/tests/helpers" HYPOTHESIS_STORAGE_DIRECTORY=/tmp/hyp \
  python -m pytest -p tensorsat_alias -p no:cacheprovider oracle/_ref/ref_tests -q -rf --timeout 300 \
  --deselect oracle/_ref/ref_tests/test_acceptance.py::test_c6_cycle_constraint_blowup_direction "$@"
