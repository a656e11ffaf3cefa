set -x
nproc; free -g; lscpu | head -20; nvidia-smi; df -h /tmp | tail -1
./tools/scatter_probe
