#!/bin/bash
# compute-sanitizer (memcheck / synccheck) on the tcgen05 prefill kernels
# (prep_tc_kernel + prefill_tc_kernel, balanced split) over a 128K context and
# on the LEAN kernels after this round's changes; logs -> gpurun_out/san2/.
O=${O:-gpurun_out/san2}
mkdir -p $O
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=_tc_kernel \
    python tools/dev/prefill_err.py 32768 > $O/san_${tool}_prefill.log 2>&1
  echo "$tool prefill rc=$?"; tail -2 $O/san_${tool}_prefill.log
  timeout 900 compute-sanitizer --tool $tool --kernel-name kns=decode_kernel \
    python tools/profile_decode.py 131072 > $O/san_${tool}_decode.log 2>&1
  echo "$tool decode rc=$?"; tail -2 $O/san_${tool}_decode.log
done
