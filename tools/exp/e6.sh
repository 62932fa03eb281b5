cd /root/repo
python tools/phases.py --cfg 4 --scenes 128 --iters 5 > gpurun_out/p4.txt 2>&1; echo "rc4=$?"
python tools/phases.py --cfg 5 --iters 5 > gpurun_out/p5.txt 2>&1; echo "rc5=$?"
tail -n 3 gpurun_out/p4.txt gpurun_out/p5.txt | cut -c1-800
