// optb_cli.cpp -- the `encode` / `decode` subcommands of the reference CLI
// (cli.cpp:61-104, option names from cli.cpp:229-243, exit codes cli.hpp:7-10)
// on the B200 drop-in library: encode/decode run on the GPU through the C++
// shim (optb/codec.hpp).  The training/bench subcommands belong to the
// reference's out-of-scope gradient-flow code and are not provided.
//
//   optb_b200 encode --mode exact128 --height 32 --width 32 [--channels 3] --out b.optb a.raw b.raw ...
//   optb_b200 decode b.optb [--out-dir DIR]
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "optb/codec.hpp"

namespace {

constexpr int kExitOk = 0, kExitUsage = 1, kExitData = 2;

struct Usage : std::runtime_error {
  using std::runtime_error::runtime_error;
};

optb::codec::CodecMode parse_mode(const std::string& name) {  // cli.cpp:15-23
  using optb::codec::CodecMode;
  if (name == "exact64") return CodecMode::ExactInt64;
  if (name == "exact128") return CodecMode::ExactInt128;
  if (name == "f64") return CodecMode::Float64Faithful;
  if (name == "lossless64") return CodecMode::LosslessOffset64;
  if (name == "lossless128") return CodecMode::LosslessOffset128;
  throw Usage("--mode: expected exact64|exact128|f64|lossless64|lossless128, got " + name);
}

uint32_t parse_u32(const std::string& flag, const std::string& v) {
  try {
    size_t used = 0;
    const unsigned long x = std::stoul(v, &used);
    if (used != v.size()) throw std::invalid_argument(v);
    return static_cast<uint32_t>(x);
  } catch (const std::exception&) {
    throw Usage(flag + ": not an unsigned integer: " + v);
  }
}

int cmd_encode(const std::vector<std::string>& args) {
  std::string mode = "exact64", out;
  uint32_t h = 0, w = 0, c = 1;
  bool has_h = false, has_w = false;
  std::vector<std::string> files;
  for (size_t i = 0; i < args.size(); ++i) {
    const std::string& a = args[i];
    auto value = [&]() -> std::string {
      if (i + 1 >= args.size()) throw Usage(a + " requires a value");
      return args[++i];
    };
    if (a == "--mode") mode = value();
    else if (a == "--height") { h = parse_u32(a, value()); has_h = true; }
    else if (a == "--width") { w = parse_u32(a, value()); has_w = true; }
    else if (a == "--channels") c = parse_u32(a, value());
    else if (a == "--out") out = value();
    else if (a.rfind("--", 0) == 0) throw Usage("unknown option " + a);
    else files.push_back(a);
  }
  if (!has_h || !has_w || out.empty() || files.empty())
    throw Usage("encode: --height, --width, --out and at least one file are required");
  const auto cm = parse_mode(mode);
  const optb::codec::ImageShape shape{h, w, c};
  std::vector<optb::codec::Image> images;
  for (const std::string& file : files) {  // cli.cpp:65-78
    std::ifstream in(file, std::ios::binary);
    if (!in) throw optb::FormatError("cannot open image file " + file);
    optb::codec::Image img;
    img.shape = shape;
    img.pixels.resize(shape.pixel_count());
    in.read(reinterpret_cast<char*>(img.pixels.data()), static_cast<std::streamsize>(img.pixels.size()));
    if (static_cast<size_t>(in.gcount()) != img.pixels.size() || in.peek() != EOF)
      throw optb::FormatError("image file " + file + " is not exactly " + std::to_string(img.pixels.size()) +
                              " bytes");
    images.push_back(std::move(img));
  }
  optb::codec::write_optb_file(out, optb::codec::encode(images, cm));
  std::cout << "wrote " << out << " (" << images.size() << " images, " << optb::codec::mode_name(cm) << ")\n";
  return kExitOk;
}

int cmd_decode(const std::vector<std::string>& args) {
  std::string input, out_dir = ".";
  for (size_t i = 0; i < args.size(); ++i) {
    if (args[i] == "--out-dir") {
      if (i + 1 >= args.size()) throw Usage("--out-dir requires a value");
      out_dir = args[++i];
    } else if (args[i].rfind("--", 0) == 0) {
      throw Usage("unknown option " + args[i]);
    } else if (input.empty()) {
      input = args[i];
    } else {
      throw Usage("decode: one input file expected");
    }
  }
  if (input.empty()) throw Usage("decode: input file required");
  const auto enc = optb::codec::read_optb_file(input);  // cli.cpp:90-104
  const auto images = optb::codec::decode(enc);
  std::filesystem::create_directories(out_dir);
  for (size_t i = 0; i < images.size(); ++i) {
    const auto path = std::filesystem::path(out_dir) / ("img_" + std::to_string(i) + ".raw");
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw optb::FormatError("cannot open output file " + path.string());
    out.write(reinterpret_cast<const char*>(images[i].pixels.data()),
              static_cast<std::streamsize>(images[i].pixels.size()));
  }
  std::cout << "decoded " << images.size() << " images from " << input << "\n";
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: optb_b200 {encode|decode} ...\n";
    return kExitUsage;
  }
  const std::string cmd = argv[1];
  const std::vector<std::string> args(argv + 2, argv + argc);
  try {
    if (cmd == "encode") return cmd_encode(args);
    if (cmd == "decode") return cmd_decode(args);
    throw Usage("unknown subcommand " + cmd);
  } catch (const Usage& e) {
    std::cerr << "usage error: " << e.what() << "\n";
    return kExitUsage;
  } catch (const optb::Error& e) {  // cli.cpp:289-300: data / format errors
    std::cerr << "error: " << e.what() << "\n";
    return kExitData;
  }
}
