# Microbenchmarks behind the scan design (profiles/r01_scatter_probe.txt, r01_access_probe.txt,
# r01_vmm_probe.txt):
#   make -C tools && /usr/local/graft/bin/gpurun --timeout 1200 -- 'bash tools/gpu_probes.sh'
nproc; free -g; nvidia-smi
./tools/scatter_probe > gpurun_out/scatter_probe.txt 2>&1
./tools/bin/fetch_probe > gpurun_out/access_probe.txt 2>&1
./tools/bin/vmm_probe > gpurun_out/vmm_probe.txt 2>&1
