#!/bin/bash
# The bounds-checked build (-DFGC_BOUNDS: device FGC_CHECK asserts trap on an
# out-of-range shared / distributed-shared / global index) under the GPU test
# suite and the sanitizer driver -- the substitute for compute-sanitizer,
# which is closed on this pool.  usage: bash tools/gpu_bounds.sh
mkdir -p gpurun_out
FGC_NVCC_FLAGS=-DFGC_BOUNDS python -c "import __graft_entry__ as g; g.build()" > gpurun_out/bounds_build.log 2>&1 || { echo build failed; tail gpurun_out/bounds_build.log; exit 1; }
FGC_NVCC_FLAGS=-DFGC_BOUNDS timeout 300 python tools/sanitize_driver.py > gpurun_out/bounds_driver.log 2>&1; echo "driver rc=$?" >> gpurun_out/bounds_driver.log
FGC_NVCC_FLAGS=-DFGC_BOUNDS timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -W ignore::DeprecationWarning > gpurun_out/bounds_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/bounds_pytest.log
grep -h "FGC_CHECK" gpurun_out/bounds_*.log | head -20
tail -2 gpurun_out/bounds_driver.log; tail -3 gpurun_out/bounds_pytest.log
