name=$1; kre=$2; shift 2
ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$kre" -c 1 -o gpurun_out/$name "$@" > gpurun_out/ncu_$name.log 2>&1
ncu -i gpurun_out/$name.ncu-rep --page raw --csv > gpurun_out/$name.csv 2>/dev/null
ncu -i gpurun_out/$name.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/${name}_src.csv 2>/dev/null
rm -f gpurun_out/$name.ncu-rep
