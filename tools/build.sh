#!/bin/bash
# rebuild the CUDA library with ptxas stats; fail loudly
PS_FORCE_BUILD=1 python -c "import __graft_entry__ as g; g.NVCC_FLAGS += ['-Xptxas','-v']; g.build_lib(); g.build_lib(debug=True)" > /tmp/build.log 2>&1
rc=$?
grep -E " error|error:" /tmp/build.log | head
grep -A2 "merge_pipe_kernelI[il]\|merge_small_kernelIi" /tmp/build.log | grep -E "Used|stack"
exit $rc
