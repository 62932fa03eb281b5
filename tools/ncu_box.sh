# run on the GPU box: full ncu capture of selected kernels, summarised to CSV
# usage: bash tools/ncu_box.sh NAME REGEX COUNT -- command...
name=$1; rx=$2; cnt=$3; shift 4
cd /root/repo; mkdir -p gpurun_out
ncu -f $NVTX --set full --import-source on --clock-control none --kernel-name-base demangled -k "regex:$rx" -c $cnt -o /tmp/$name "$@" > gpurun_out/$name.log 2>&1
ncu -i /tmp/$name.ncu-rep --page raw --csv > gpurun_out/$name.raw.csv 2>/dev/null
for i in $(seq 0 $((cnt-1))); do python tools/ncu_lines.py /tmp/$name.ncu-rep --launch $i --top 40 > gpurun_out/$name.lines$i.txt 2>&1; done
