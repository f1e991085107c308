// tt_ws_w1.cu -- instantiation of the warp-specialised contraction kernel, tile ws80x160x16.
#include "tt_contract_ws.cuh"

namespace tt { namespace ws { using Cfg_w1 = WCfg<80, 160, 16, 2, 4, 6, 1>; } }
TT_WS_DEFINE(w1, ws::Cfg_w1, "ws80x160x16")
