set -x
nvidia-smi; nproc; lscpu | grep -E "Model name|^CPU\(s\)|Thread|Socket"; free -g | head -2
ls -d /root/reference 2>&1; ls baseline 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/intpipe tools/microbench/intpipe.cu && ./tools/microbench/intpipe
