# which of the two changes breaks the C4 n=32 norm: persistent kernels or split sign flips
for e in "QCS_PERSIST=0 QCS_JIT_SPLIT_SIGNS=0" "QCS_PERSIST=0 QCS_JIT_SPLIT_SIGNS=1" "QCS_PERSIST=1 QCS_JIT_SPLIT_SIGNS=0" "QCS_PERSIST=1 QCS_JIT_SPLIT_SIGNS=1"; do
  env $e timeout 300 python tools/norm_check.py 32 4 2>&1 | tail -1
done
env QCS_PERSIST=1 QCS_JIT_SPLIT_SIGNS=0 timeout 300 python tools/norm_check.py 30 6 2>&1 | tail -1
env QCS_PERSIST=1 QCS_JIT_SPLIT_SIGNS=0 timeout 300 python tools/norm_check.py 28 8 2>&1 | tail -1
