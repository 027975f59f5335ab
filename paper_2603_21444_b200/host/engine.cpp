// EventTimeline serialisation (reference engine.cpp:12-41): same names, same
// key order, numbers printed the way nlohmann::json dumps them (integers as
// integers, doubles in the shortest form that round-trips).
#include "spgsim/engine.hpp"

#include <charconv>
#include <cmath>

namespace spgsim {

const char* operand_name(Operand o) { return o == Operand::A ? "A" : "B"; }

const char* event_name(EventType t) {
    switch (t) {
        case EventType::enqueue_request: return "enqueue-request";
        case EventType::serve_request: return "serve-request";
        case EventType::transfer_complete: return "transfer-complete";
        case EventType::allgather_complete: return "allgather-complete";
        case EventType::compute_complete: return "compute-complete";
    }
    return "?";
}

namespace {
void put_double(std::string& out, double v) {
    if (!std::isfinite(v)) {
        out += "null";
        return;
    }
    char buf[64];
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    std::string s(buf, r.ptr);
    // nlohmann prints integral doubles with a trailing ".0"
    if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
    out += s;
}
void put_int(std::string& out, std::int64_t v) {
    char buf[32];
    auto r = std::to_chars(buf, buf + sizeof(buf), v);
    out.append(buf, r.ptr);
}
}  // namespace

std::string EventTimeline::to_jsonl() const {
    std::string out;
    for (const auto& e : events) {
        out += "{\"type\":\"";
        out += event_name(e.type);
        out += "\",\"actors\":[";
        put_int(out, e.src);
        out += ",";
        put_int(out, e.dst);
        out += "],\"round\":";
        put_int(out, e.round);
        out += ",\"t_start\":";
        put_double(out, e.t_start);
        out += ",\"t_end\":";
        put_double(out, e.t_end);
        out += ",\"bytes\":";
        put_int(out, e.bytes);
        out += ",\"operand\":\"";
        out += operand_name(e.operand);
        out += "\",\"link\":\"";
        out += link_name(e.link);
        out += "\",\"nnz\":";
        put_int(out, e.nnz);
        out += "}\n";
    }
    return out;
}

}  // namespace spgsim
