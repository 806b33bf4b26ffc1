# TEST INFRASTRUCTURE ONLY.  Compiles the reference's own hot-path sources IN
# PLACE from /root/reference (nothing is copied into this repo) into
# oracle/_ref/libhegmm_refcore.so, and oracle/ref_shim.cpp + the CPU oracle
# into oracle/_ref/libhegmm_ref.so.  oracle/_ref/ is
# git-ignored but travels to the GPU box with the gpurun snapshot.
CXX ?= g++
REF ?= /root/reference/proj
HERE := $(dir $(abspath $(lastword $(MAKEFILE_LIST))))
OUT := $(HERE)_ref
SRCS := $(REF)/src/matrix.cpp $(REF)/src/backend.cpp $(REF)/src/lintrans.cpp $(REF)/src/algorithms.cpp \
        $(REF)/src/costmodel.cpp
# costmodel.cpp includes <json.hpp> (nlohmann); the image carries a copy under cudnn_frontend
JSON_INC ?= $(firstword $(wildcard /opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann))

# Two libraries, so the reference-side binding (integration/) links the
# reference's code only and never the test checkers:
#   _ref/libhegmm_refcore.so  the reference's own sources, nothing else
#   _ref/libhegmm_ref.so      ref_shim.cpp + the CPU oracle (test infrastructure), on top of it
all: $(OUT)/libhegmm_ref.so

$(OUT)/libhegmm_refcore.so: $(SRCS)
	mkdir -p $(OUT)
	$(CXX) -O2 -std=c++20 -fPIC -shared -I$(REF)/include -I$(JSON_INC) -o $@ $(SRCS) -lpthread

$(OUT)/libhegmm_ref.so: $(OUT)/libhegmm_refcore.so $(HERE)ref_shim.cpp $(HERE)bfv_oracle.cpp $(HERE)bfv_oracle.h
	$(CXX) -O2 -std=c++20 -fPIC -shared -I$(REF)/include -I$(HERE) -I$(JSON_INC) -o $@ \
	    $(HERE)ref_shim.cpp $(HERE)bfv_oracle.cpp -L$(OUT) -l:libhegmm_refcore.so -Wl,-rpath,'$$ORIGIN' -lpthread
.PHONY: all
