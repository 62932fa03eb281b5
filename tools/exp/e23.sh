cd /root/repo
for i in 1 2; do
echo new; python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-40
echo old; PDF_LIB_PATH=tools/exp/lib_37ca7cf.so python tools/timeline.py --cfg 3 2>&1 | tail -1 | cut -c1-40
done
PDF_LIB_PATH=tools/exp/lib_37ca7cf.so python tools/timeline.py --cfg 3 2>&1 | tail -13 | head -10
