#!/bin/bash
# compute-sanitizer (memcheck / synccheck / racecheck) on the fused decode
# kernel (4 launches: 2 warm-up misses, a miss, a hit) at 128K and 142K;
# logs -> profiles/r02_sanitizer/.
mkdir -p gpurun_out
for tool in memcheck synccheck racecheck; do
  for n in 131072 142336; do
    timeout 600 compute-sanitizer --tool $tool --kernel-name kns=decode_kernel \
      python tools/profile_decode.py $n > gpurun_out/san_${tool}_${n}.log 2>&1
    echo "$tool $n rc=$?"; tail -2 gpurun_out/san_${tool}_${n}.log
  done
done
