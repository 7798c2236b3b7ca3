# mkvar.sh NAME "FLAGS": builds build_probe/libbl_NAME.so with decode mode 2 compiled with FLAGS
set -e
cd /root/repo/paper_2101_05600_b200/csrc
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr $2 -DDK_MODE=0 -c decode_kernel.cu -o /root/repo/build_probe/decode_m0_$1.o
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared /root/repo/build_probe/decode_m0_$1.o build/decode_m1.o build/decode_m2.o build/decode_m3.o build/decode_m4.o build/capi.o build/gemm_tcgen05.o build/encoder.o build/decoder_net.o -o /root/repo/build_probe/libbl_$1.so
