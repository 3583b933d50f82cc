"""paper_1409_2802_b200 -- B200-native far-field passes of arXiv 1409.2802 (kernid).

Native libraries (built in-tree by build.py / __graft_entry__.build()):
  libkernid_cuda.so  sm_100a kernels behind the C-ABI include/kernid_cuda.h
  libkernid_host.so  C++ mirror of the reference kernid:: API (include/kernid_b200.hpp)
"""
__all__ = ["build"]
