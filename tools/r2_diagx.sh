#!/bin/bash
mkdir -p gpurun_out/dx
for r in 1 2; do for v in old new new2; do echo -n "$v: "; ./tools/ubench_diag_$v gpurun_out/dx/$v.bin; done; done
for v in new new2; do cmp gpurun_out/dx/old.bin gpurun_out/dx/$v.bin && echo "$v bitwise same"; cmp gpurun_out/dx/old.bin.tiny gpurun_out/dx/$v.bin.tiny && echo "$v tiny bitwise same"; done
