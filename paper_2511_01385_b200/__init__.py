"""B200-native rdFFT hot path (arXiv 2511.01385): in-place real-domain FFT,
packed products and the fused block-circulant (BCA) layer, as hand-written
CUDA for sm_100a behind the C-ABI library librdfft.so (include/rdfft.h)."""
