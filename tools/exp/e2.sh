cd /root/repo
echo X1; bash tools/skip_sweep.sh --cfg 2
echo X0; PDF_FWD_X=0 bash tools/skip_sweep.sh --cfg 2
