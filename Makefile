# C++ side of hookcc-b200.
#   make lib       libhookcc_cuda.so (nvcc, sm_100a)       -> paper_1612_01178_b200/lib/
#   make cc        the `cc` CLI on the B200 library         -> bin/cc
#   make reftests  the REFERENCE's own test sources (compiled in place from
#                  /root/reference/proj/tests against this repo's headers; not
#                  copied)                                  -> tests/cpp/_bin/
#   make oracle    CPU checkers                             -> oracle/
# Built artefacts are git-ignored but travel to the GPU box with the repo.
ROOT := $(dir $(abspath $(lastword $(MAKEFILE_LIST))))
REF_TESTS ?= /root/reference/proj/tests
JSON_INC ?= $(shell python3 -c "import os,site;print(next((os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann') for p in site.getsitepackages() if os.path.exists(os.path.join(p,'include/cudnn_frontend/thirdparty/nlohmann/json.hpp'))),''))")
CXX ?= g++
CXXFLAGS ?= -std=c++20 -O2 -Wall -Wno-unused-variable
INC := -I$(ROOT)include -I$(JSON_INC)
LIBDIR := $(ROOT)paper_1612_01178_b200/lib
LDLIBS := -L$(LIBDIR) -lhookcc_cuda -Wl,-rpath,$(LIBDIR) -pthread
HDRS := $(wildcard $(ROOT)include/hookcc/*.hpp) $(ROOT)include/hookcc_c.h
LIBSO := $(LIBDIR)/libhookcc_cuda.so

all: lib cc reftests apitests oracle

lib:
	python3 -m paper_1612_01178_b200.build

$(LIBSO): lib

cc: $(ROOT)bin/cc
$(ROOT)bin/cc: $(ROOT)tools/cc_main.cpp $(HDRS) | $(LIBSO)
	@mkdir -p $(ROOT)bin
	$(CXX) $(CXXFLAGS) $(INC) -o $@ $< $(LDLIBS)

BIN := $(ROOT)tests/cpp/_bin
SHIM := -I$(ROOT)tests/cpp/shim
UNIT_SRCS := $(wildcard $(REF_TESTS)/test_*.cpp)

reftests:
	@if [ -d "$(REF_TESTS)" ]; then \
	  $(MAKE) -f $(ROOT)Makefile $(BIN)/unit_tests $(BIN)/acceptance; \
	else echo "reference tests absent: using prebuilt $(BIN)"; fi

$(BIN)/unit_tests: $(UNIT_SRCS) $(ROOT)tests/cpp/shim/catch_main.cpp $(HDRS) | $(LIBSO)
	@mkdir -p $(BIN)
	$(CXX) $(CXXFLAGS) $(INC) $(SHIM) -o $@ $(UNIT_SRCS) $(ROOT)tests/cpp/shim/catch_main.cpp $(LDLIBS)

$(BIN)/acceptance: $(REF_TESTS)/acceptance.cpp $(HDRS) | $(LIBSO)
	@mkdir -p $(BIN)
	$(CXX) $(CXXFLAGS) $(INC) -DFIXTURE_DIR=\"$(ROOT)tests/golden/fixtures\" -o $@ $< $(LDLIBS)

# B200-only API additions (own sources, no reference needed)
apitests: $(BIN)/api_extras
$(BIN)/api_extras: $(ROOT)tests/cpp/test_api_extras.cpp $(ROOT)tests/cpp/shim/catch_main.cpp $(HDRS) $(ROOT)include/hookcc/verify.hpp | $(LIBSO)
	@mkdir -p $(BIN)
	$(CXX) $(CXXFLAGS) $(INC) $(SHIM) -o $@ $(ROOT)tests/cpp/test_api_extras.cpp $(ROOT)tests/cpp/shim/catch_main.cpp $(LDLIBS)

oracle:
	$(MAKE) -C $(ROOT)oracle

.PHONY: all lib cc reftests apitests oracle
