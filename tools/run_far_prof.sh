python tools/asm_only.py 2 1.0 1 > gpurun_out/asm2.log 2>&1; tail -2 gpurun_out/asm2.log
ncu --set full --import-source on --clock-control none --kernel-name-base demangled --kernel-name regex:"k_far<\(int\)4, \(int\)3>" -c 1 -o gpurun_out/prof_far43 -f python tools/asm_only.py 2 1.0 1 > gpurun_out/ncu_far43.log 2>&1; echo rc=$?
